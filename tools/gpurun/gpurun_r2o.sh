cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { name=$1; shift; timeout 300 python bench.py --no-cpu-baseline "$@" > gpurun_out/o_$name.json 2> gpurun_out/o_$name.err
  python - gpurun_out/o_$name.json "$name" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), d["stage_ms_last"], "commit", d["step_breakdown"]["commit_ms"], d["gpu_launches"])
except Exception as e: print(sys.argv[2], "ERR", e)
PY
}
run wl2
run wl2b
run wl5 --workload 5
run wl1 --workload 1
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/o_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/o_pytest.log
