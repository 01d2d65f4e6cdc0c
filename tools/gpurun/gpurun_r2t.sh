cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
SKV_PROBE_SPLIT=0 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_golden.py tests/test_gpu_configs.py tests/test_gpu_edges.py -x -q -p no:cacheprovider > gpurun_out/t_pytest_split0.log 2>&1; echo "split0 rc=$?"; tail -1 gpurun_out/t_pytest_split0.log
SKV_PROBE_SPLIT=32 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_configs.py -x -q -p no:cacheprovider > gpurun_out/t_pytest_split32.log 2>&1; echo "split32 rc=$?"; tail -1 gpurun_out/t_pytest_split32.log
timeout 900 python -m pytest tests/test_gpu_scale.py tests/test_gpu_graphs.py -x -q -p no:cacheprovider > gpurun_out/t_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/t_pytest.log
for w in 2 6 4 5; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/t_wl$w.json 2>/dev/null
python - gpurun_out/t_wl$w.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), d["stage_ms_last"])
PY
done
