cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_golden.py -x -q -p no:cacheprovider > gpurun_out/y_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/y_pytest.log
T="tests/test_gpu_graphs.py tests/test_gpu_golden.py::test_config1_golden tests/test_gpu_parity.py::test_parity_b16_w32 tests/test_gpu_prefetch.py::test_step_host_pipeline_parity"
timeout 1200 compute-sanitizer --tool memcheck --leak-check no --target-processes all --print-limit 30 python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/y_san_memcheck.log 2>&1
echo "memcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/y_san_memcheck.log | tail -2 | tr '\n' ' ')"
timeout 300 python tools/config1_latency.py > gpurun_out/y_cfg1.json 2>&1; cat gpurun_out/y_cfg1.json
