cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_hash_scan16$" -s 3 -c 1 -o gpurun_out/hs_full python tools/hs_probe.py > gpurun_out/hs_ncu.log 2>&1; echo "ncu rc=$?"
