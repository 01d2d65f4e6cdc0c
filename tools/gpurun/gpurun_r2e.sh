cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_golden.py tests/test_gpu_parity.py -x -q -p no:cacheprovider > gpurun_out/e_pytest1.log 2>&1; echo "pytest1 rc=$?"; tail -15 gpurun_out/e_pytest1.log
timeout 300 python tools/small_timeline.py > gpurun_out/e_small_timeline.txt 2>&1; cat gpurun_out/e_small_timeline.txt | tail -3
SKV_GRAPHS=0 timeout 300 python tools/small_timeline.py > gpurun_out/e_small_timeline_nograph.txt 2>&1; cat gpurun_out/e_small_timeline_nograph.txt | tail -3
timeout 300 python tools/config1_latency.py > gpurun_out/e_cfg1_latency.json 2>&1; cat gpurun_out/e_cfg1_latency.json
for v in "wl1 --workload 1" "wl1np --workload 1 --no-pipeline" "wl5 --workload 5" "wl5np --workload 5 --no-pipeline" "wl2 --workload 2"; do set -- $v; name=$1; shift
  timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/e_$name.json 2> gpurun_out/e_$name.err
  python - gpurun_out/e_$name.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]/1e9,4), d["ms_per_step"], "e2e", round(d["e2e"]["value"]/1e9,4), d["stage_ms_last"], d["roofline"]["frac"], d["gpu_launches"])
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
timeout 1500 python -m pytest tests -x -q -m gpu -p no:cacheprovider > gpurun_out/e_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/e_pytest.log
