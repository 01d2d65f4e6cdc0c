cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
run() { name=$1; shift; env "$@" timeout 300 python bench.py --no-cpu-baseline > gpurun_out/n_$name.json 2> gpurun_out/n_$name.err
  python - gpurun_out/n_$name.json "$name" <<'PY'
import json,sys
try:
    d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
    print(sys.argv[2], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), "hs", d["stage_ms_last"]["hash_scan_ms"], "probe", d["stage_ms_last"]["chain_probe_ms"], "commit", d["step_breakdown"]["commit_ms"], "ep", d["stage_ms_last"]["epoch_ms"])
except Exception as e: print(sys.argv[2], "ERR", e)
PY
}
run base SKV_X=0
run pf4c111 SKV_COMMIT_SMS=111
run pf3 SKV_H16_PF_FRAC=3
run pf3c99 SKV_H16_PF_FRAC=3 SKV_COMMIT_SMS=99
run pf2c74 SKV_H16_PF_FRAC=2 SKV_COMMIT_SMS=74
run pf3c111 SKV_H16_PF_FRAC=3 SKV_COMMIT_SMS=111
run pf5 SKV_H16_PF_FRAC=5
