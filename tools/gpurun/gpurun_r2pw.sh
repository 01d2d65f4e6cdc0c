cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline $BARGS > gpurun_out/pw_$name.json 2> gpurun_out/pw_$name.err
  python - gpurun_out/pw_$name.json "$name" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), "hs", d["stage_ms_last"]["hash_scan_ms"], "probe", d["stage_ms_last"]["chain_probe_ms"], "commit", d["step_breakdown"]["commit_ms"])
except Exception as e: print(sys.argv[2], "ERR", e)
PY
}
BARGS="" run w8 SKV_H16_PF_WARPS=8
BARGS="" run w10 SKV_H16_PF_WARPS=10
BARGS="" run w12 SKV_H16_PF_WARPS=12
BARGS="" run w6 SKV_H16_PF_WARPS=6
BARGS="" run w8b SKV_H16_PF_WARPS=8
BARGS="--workload 6" run w8_6 SKV_H16_PF_WARPS=8
BARGS="--workload 6" run w12_6 SKV_H16_PF_WARPS=12
