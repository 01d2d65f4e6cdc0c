cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest7.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench7.json 2> gpurun_out/bench7.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches7.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch7.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_chain_probe|k_record_finish" -s 4 -c 2 -o gpurun_out/prof7 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full7.log 2>&1
