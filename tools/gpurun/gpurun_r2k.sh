cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_golden.py tests/test_gpu_parity.py tests/test_gpu_rule_groups.py tests/test_gpu_prefetch.py tests/test_gpu_edges.py tests/test_gpu_configs.py "tests/test_gpu_scale.py::test_scale_config2_full_batches" -x -q -p no:cacheprovider > gpurun_out/k_pytest1.log 2>&1; echo "pytest1 rc=$?"; tail -3 gpurun_out/k_pytest1.log
timeout 300 python tools/hs_probe.py > gpurun_out/k_hs_probe.txt 2>&1; tail -5 gpurun_out/k_hs_probe.txt
timeout 300 python tools/config1_latency.py > gpurun_out/k_cfg1_latency.json 2>&1; cat gpurun_out/k_cfg1_latency.json
for v in "wl1 --workload 1" "wl1f --workload 1 --fused-step 1" "wl5 --workload 5" "wl2 --workload 2"; do set -- $v; name=$1; shift
  timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/k_$name.json 2> gpurun_out/k_$name.err
  python - gpurun_out/k_$name.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]/1e9,4), d["ms_per_step"], "e2e", round(d["e2e"]["value"]/1e9,4), d["stage_ms_last"], round(d["roofline"]["frac"],4), d["roofline"]["avg_launch_ms"])
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/k_cfg1_launches.csv python tools/config1_latency.py --reps 3 > /dev/null 2>&1; echo "ncu rc=$?"
timeout 600 compute-sanitizer --tool racecheck --print-limit 20 python -m pytest tests/test_gpu_golden.py::test_config1_golden tests/test_gpu_parity.py::test_parity_b16_w32 -x -q -p no:cacheprovider > gpurun_out/k_racecheck.log 2>&1; echo "racecheck $(grep -E 'RACECHECK SUMMARY|passed' gpurun_out/k_racecheck.log | tr '\n' ' ')"
timeout 600 compute-sanitizer --tool synccheck --print-limit 20 python -m pytest tests/test_gpu_golden.py::test_config1_golden tests/test_gpu_parity.py::test_parity_b16_w32 -x -q -p no:cacheprovider > gpurun_out/k_synccheck.log 2>&1; echo "synccheck $(grep -E 'ERROR SUMMARY|passed' gpurun_out/k_synccheck.log | tr '\n' ' ')"
