cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/small_timeline.py > gpurun_out/d_small_timeline.txt 2>&1; echo "timeline rc=$?"; cat gpurun_out/d_small_timeline.txt
timeout 300 python tools/config1_latency.py > gpurun_out/d_cfg1_latency.json 2>&1; cat gpurun_out/d_cfg1_latency.json
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/d_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/d_pytest.log
timeout 300 python bench.py --workload 1 --no-cpu-baseline > gpurun_out/d_wl1.json 2>/dev/null
timeout 300 python bench.py --workload 5 --no-cpu-baseline > gpurun_out/d_wl5.json 2>/dev/null
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/d_wl2.json 2>/dev/null
timeout 900 python bench.py --workload 3 --no-cpu-baseline > gpurun_out/d_wl3.json 2> gpurun_out/d_wl3.err; echo "wl3 rc=$?"
for f in gpurun_out/d_wl*.json; do python - "$f" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]/1e9,4), d["ms_per_step"], d["stage_ms_last"], d["roofline"]["frac"])
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
timeout 900 compute-sanitizer --tool initcheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py::test_parity_b16_w32 tests/test_gpu_golden.py::test_config1_golden -x -q -p no:cacheprovider > gpurun_out/d_initcheck.log 2>&1
echo "initcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/d_initcheck.log | tail -2 | tr '\n' ' ')"
timeout 900 compute-sanitizer --tool racecheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py::test_parity_b16_w32 tests/test_gpu_golden.py::test_config1_golden -x -q -p no:cacheprovider > gpurun_out/d_racecheck.log 2>&1
echo "racecheck rc=$? $(grep -E 'RACECHECK SUMMARY|passed|failed' gpurun_out/d_racecheck.log | tail -2 | tr '\n' ' ')"
timeout 900 compute-sanitizer --tool synccheck --target-processes all --print-limit 20 python -m pytest tests/test_gpu_parity.py::test_parity_b16_w32 tests/test_gpu_golden.py::test_config1_golden -x -q -p no:cacheprovider > gpurun_out/d_synccheck.log 2>&1
echo "synccheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/d_synccheck.log | tail -2 | tr '\n' ' ')"
