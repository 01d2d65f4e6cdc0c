cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29541 bench.py --gpus 2 --workload 6 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mg_wl6_n2.json 2> gpurun_out/mg_wl6_n2.err; echo "wl6 n2 rc=$?"; tail -c 900 gpurun_out/mg_wl6_n2.json; echo
timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29542 bench.py --gpus 4 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/mg_wl2_n4.json 2> gpurun_out/mg_wl2_n4.err; echo "wl2 n4 rc=$?"; tail -c 600 gpurun_out/mg_wl2_n4.json; echo
tail -3 gpurun_out/mg_wl2_n4.err
