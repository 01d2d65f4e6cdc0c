cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_graphs.py tests/test_gpu_prefetch.py tests/test_gpu_parity.py tests/test_bench_contract.py -x -q -p no:cacheprovider > gpurun_out/m_pytest1.log 2>&1; echo "pytest1 rc=$?"; tail -15 gpurun_out/m_pytest1.log
for v in "wl2 --workload 2" "wl2s --workload 2 --fused-step 0" "wl1 --workload 1" "wl1s --workload 1 --fused-step 0" "wl5 --workload 5" "wl5s --workload 5 --fused-step 0"; do set -- $v; name=$1; shift
  timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/m_$name.json 2> gpurun_out/m_$name.err
  python - gpurun_out/m_$name.json <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[1], round(d["value"]/1e9,4), d["ms_per_step"], "e2e", round(d["e2e"]["value"]/1e9,4), d["stage_ms_last"], round(d["roofline"]["frac"],4))
except Exception as e: print(sys.argv[1], "ERR", e)
PY
done
tail -3 gpurun_out/m_wl2.err
