cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_facade.py -q -p no:cacheprovider > gpurun_out/l_pytest1.log 2>&1; echo "pytest1 rc=$?"; tail -30 gpurun_out/l_pytest1.log
