cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"k_epoch" --csv --log-file gpurun_out/c4e_launches.csv python bench.py --workload 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4e.log 2>&1; echo "ncu rc=$?"
