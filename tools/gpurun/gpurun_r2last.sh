cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -q -m gpu -p no:cacheprovider > gpurun_out/last_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/last_pytest.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/last_smoke.log 2>&1; echo "smoke rc=$?"; cat gpurun_out/last_smoke.log
timeout 900 python bench.py > gpurun_out/last_bench.json 2> gpurun_out/last_bench.err; echo "bench rc=$?"
python - gpurun_out/last_bench.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), "frac", round(d["roofline"]["frac"],4), d["cpu_baseline"]["value"], d["clocks"])
PY
