cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/i_smi.txt 2>&1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider --durations=15 > gpurun_out/i_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/i_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/i_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py > gpurun_out/i_bench.json 2> gpurun_out/i_bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/i_ref.json 2> gpurun_out/i_ref.err; echo "ref rc=$?"
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/i_bench_n2.json 2> gpurun_out/i_bench_n2.err; echo "n2 rc=$?"; tail -c 600 gpurun_out/i_bench_n2.json
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --gpus 2 --impl reference --steps 2 --warmup 1 > gpurun_out/i_ref_n2.json 2> gpurun_out/i_ref_n2.err; echo "ref n2 rc=$?"; tail -c 300 gpurun_out/i_ref_n2.json
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/i_launches.csv python bench.py --steps 2 --warmup 1 --no-cpu-baseline > gpurun_out/i_ncu_launch.log 2>&1; echo "ncu launches rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"^(k_hash_scan16|k_chain_probe|k_commit)$" -s 30 -c 4 -o gpurun_out/i_full python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/i_ncu_full.log 2>&1; echo "ncu full rc=$?"
cat gpurun_out/i_bench.json gpurun_out/i_ref.json
