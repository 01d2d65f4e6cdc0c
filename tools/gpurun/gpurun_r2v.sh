cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline $BARGS > gpurun_out/v_$name.json 2> gpurun_out/v_$name.err
  python - gpurun_out/v_$name.json "$name" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), "hs", d["stage_ms_last"]["hash_scan_ms"], "probe", d["stage_ms_last"]["chain_probe_ms"], "commit", d["step_breakdown"]["commit_ms"])
except Exception as e: print(sys.argv[2], "ERR", e)
PY
}
BARGS="" run w8 SKV_H16_PF_WARPS=8
BARGS="" run w0 SKV_H16_PF_WARPS=0
BARGS="" run w4 SKV_H16_PF_WARPS=4
BARGS="" run w16 SKV_H16_PF_WARPS=16
BARGS="--workload 6" run w8_6 SKV_H16_PF_WARPS=8
BARGS="--workload 6" run w0_6 SKV_H16_PF_WARPS=0
BARGS="--workload 5" run w8_5 SKV_H16_PF_WARPS=8
BARGS="--workload 5" run w0_5 SKV_H16_PF_WARPS=0
timeout 600 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_scale.py::test_scale_config2_full_batches -x -q -p no:cacheprovider > gpurun_out/v_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/v_pytest.log
