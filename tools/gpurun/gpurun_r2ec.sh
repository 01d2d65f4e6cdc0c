cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_graphs.py "tests/test_gpu_scale.py::test_scale_config4_long_context_tiered" "tests/test_gpu_scale.py::test_scale_config5_adversarial_mix" -x -q -p no:cacheprovider > gpurun_out/ec_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/ec_pytest.log
for w in 4 2 5; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/ec_wl$w.json 2>/dev/null
python - gpurun_out/ec_wl$w.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "epoch avg", d["step_breakdown"]["epoch_ms"], "last", d["stage_ms_last"]["epoch_ms"])
PY
done
