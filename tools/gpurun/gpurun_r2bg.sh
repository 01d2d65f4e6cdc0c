cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -x -p no:cacheprovider > gpurun_out/bg_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/bg_pytest.log
for w in 1 5 2; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/bg_wl$w.json 2>/dev/null
python - gpurun_out/bg_wl$w.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), "commit", d["step_breakdown"]["commit_ms"])
PY
done
