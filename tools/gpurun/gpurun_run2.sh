cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu > gpurun_out/pytest2.log 2>&1
timeout 300 python __graft_entry__.py > gpurun_out/smoke2.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench2.json 2> gpurun_out/bench2.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches2.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch2.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_hash_scan -s 2 -c 1 -o gpurun_out/prof_hs2 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full2.log 2>&1
ls -la gpurun_out
