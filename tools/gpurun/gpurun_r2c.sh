cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_rule_groups.py tests/test_gpu_golden.py tests/test_gpu_facade.py tests/test_gpu_prefetch.py tests/test_gpu_parity.py tests/test_gpu_scale.py::test_scale_config2_full_batches -q -p no:cacheprovider > gpurun_out/c_pytest.log 2>&1
echo "pytest rc=$?"; tail -3 gpurun_out/c_pytest.log
for v in "pipe" "nopipe --no-pipeline"; do set -- $v; name=$1; shift
  timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/c_bench_$name.json 2> gpurun_out/c_bench_$name.err
done
for f in 2 8; do SKV_H16_PF_FRAC=$f timeout 300 python bench.py --no-cpu-baseline > gpurun_out/c_bench_pf$f.json 2>/dev/null; done
for f in gpurun_out/c_bench_*.json; do python - "$f" <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]/1e9,3), d["ms_per_step"], d["stage_ms_last"], d["step_breakdown"]["commit_ms"])
PY
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/c_cfg1_launches.csv python tools/config1_latency.py --reps 3 > gpurun_out/c_cfg1_ncu.log 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c_wl5_launches.csv python bench.py --workload 5 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/c_wl5_ncu.log 2>&1
echo done
T="tests/test_gpu_parity.py::test_parity_b16_w32 tests/test_gpu_golden.py::test_config1_golden tests/test_gpu_rule_groups.py::test_rule_groups_parity"
timeout 900 compute-sanitizer --tool racecheck --target-processes all --print-limit 50 python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/c_racecheck.log 2>&1
echo "racecheck rc=$? $(grep -E 'RACECHECK SUMMARY|passed|failed' gpurun_out/c_racecheck.log | tail -2 | tr '\n' ' ')"
timeout 900 compute-sanitizer --tool initcheck --target-processes all --print-limit 50 python -m pytest tests/test_gpu_parity.py::test_parity_b16_w32 tests/test_gpu_golden.py::test_config1_golden -x -q -p no:cacheprovider > gpurun_out/c_initcheck.log 2>&1
echo "initcheck rc=$? $(grep -E 'ERROR SUMMARY|passed|failed' gpurun_out/c_initcheck.log | tail -2 | tr '\n' ' ')"
timeout 600 python bench.py --workload 3 --no-cpu-baseline > gpurun_out/c_wl3.json 2> gpurun_out/c_wl3.err; echo "wl3 rc=$?"; tail -2 gpurun_out/c_wl3.err
nvidia-smi --query-gpu=memory.total,memory.used --format=csv
