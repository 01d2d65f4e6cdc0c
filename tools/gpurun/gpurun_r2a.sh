cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/a_smi.txt 2>&1
timeout 2400 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=30 > gpurun_out/a_pytest.log 2>&1
echo "pytest rc=$?"
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/a_smoke.log 2>&1
echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/a_bench.json 2> gpurun_out/a_bench.err
echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/a_ref.json 2> gpurun_out/a_ref.err
echo "ref rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/a_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/a_ncu_launch.log 2>&1
echo "ncu rc=$?"
tail -3 gpurun_out/a_pytest.log; cat gpurun_out/a_bench.json gpurun_out/a_ref.json
