cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_prefetch.py tests/test_gpu_graphs.py tests/test_bench_contract.py -x -q -p no:cacheprovider > gpurun_out/q_pytest.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/q_pytest.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/q_wl2_$i.json 2> gpurun_out/q_wl2_$i.err
python - gpurun_out/q_wl2_$i.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), d["config"]["pipeline"])
PY
done
