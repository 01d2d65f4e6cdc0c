cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_hash_scan$" -s 40 -c 1 -o gpurun_out/c4_hs python bench.py --workload 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c4_ncu.log 2>&1; echo "ncu rc=$?"; tail -3 gpurun_out/c4_ncu.log
