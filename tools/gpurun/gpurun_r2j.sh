cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_rule_groups.py tests/test_gpu_prefetch.py tests/test_gpu_edges.py tests/test_gpu_configs.py "tests/test_gpu_scale.py::test_scale_config5_adversarial_mix" -x -q -p no:cacheprovider > gpurun_out/j_pytest1.log 2>&1; echo "pytest1 rc=$?"; tail -3 gpurun_out/j_pytest1.log
timeout 300 python tools/config1_latency.py > gpurun_out/j_cfg1_latency.json 2>&1; cat gpurun_out/j_cfg1_latency.json
for v in "wl1 --workload 1" "wl1f --workload 1 --fused-step 1" "wl5 --workload 5" "wl5f --workload 5 --fused-step 1" "wl2 --workload 2"; do set -- $v; name=$1; shift
  timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/j_$name.json 2> gpurun_out/j_$name.err
  python - gpurun_out/j_$name.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]/1e9,4), d["ms_per_step"], "e2e", round(d["e2e"]["value"]/1e9,4), d["stage_ms_last"], round(d["roofline"]["frac"],4))
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/j_cfg1_launches.csv python tools/config1_latency.py --reps 3 > /dev/null 2>&1; echo "ncu rc=$?"
