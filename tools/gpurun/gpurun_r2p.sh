cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
bash tools/ab.sh h1 h2 h1 h2 "h1:--workload 5" "h2:--workload 5"
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_edges.py tests/test_gpu_prefetch.py tests/test_gpu_graphs.py tests/test_gpu_scale.py -x -q -p no:cacheprovider > gpurun_out/p_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/p_pytest.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"^k_chain_probe$" -s 3 -c 3 --csv --log-file gpurun_out/p_probe.csv python bench.py --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1; echo "ncu rc=$?"; grep -E "gpu__time_duration|dram__bytes_read" gpurun_out/p_probe.csv | awk -F'","' '{print $5, $(NF-2), $NF}' | head
