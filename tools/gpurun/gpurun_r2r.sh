cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/r_pytest.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r_pytest.log
