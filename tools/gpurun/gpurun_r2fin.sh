cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/fin_smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=12 > gpurun_out/fin_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/fin_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/fin_ref.json 2> gpurun_out/fin_ref.err; echo "ref rc=$?"
for w in 1 3 4 5 6; do timeout 900 python bench.py --workload $w > gpurun_out/fin_wl$w.json 2> gpurun_out/fin_wl$w.err; echo "wl$w rc=$?"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/fin_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(k_chain_probe|k_commit)$" -s 10 -c 2 -o gpurun_out/fin_full python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu_full.log 2>&1; echo "ncu full rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^k_hash_scan16$" -c 1 -o gpurun_out/fin_hs16 python tools/hs_probe.py > gpurun_out/fin_ncu_hs16.log 2>&1; echo "ncu hs16 rc=$?"
cat gpurun_out/fin_bench.json
