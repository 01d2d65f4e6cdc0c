cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/pytest5.log 2>&1
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench5.json 2> gpurun_out/bench5.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/launches5.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_launch5.log 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_hash_scan|k_chain_probe|k_commit|k_record" -s 8 -c 4 -o gpurun_out/prof5 python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/ncu_full5.log 2>&1
