cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_bench_contract.py tests/test_gpu_prefetch.py::test_step_host_pipeline_parity -q -p no:cacheprovider > gpurun_out/val_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/val_pytest.log
for w in 1 5 2; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/val_wl$w.json 2>gpurun_out/val_wl$w.err
python - gpurun_out/val_wl$w.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), d["config"]["pipeline"][-60:])
PY
done
