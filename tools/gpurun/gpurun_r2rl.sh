cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
T="tests/test_gpu_parity.py tests/test_gpu_attack.py tests/test_gpu_scale.py::test_scale_config5_adversarial_mix tests/test_gpu_scale.py::test_scale_config4_long_context_tiered tests/test_gpu_graphs.py tests/test_gpu_labels.py"
timeout 900 python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/rl_pytest.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/rl_pytest.log
cp paper_2508_08438_b200/libsafekv_b200.so /tmp/lib.orig; cp tools/gpurun/tmp_rs1/libsafekv_b200.so paper_2508_08438_b200/libsafekv_b200.so
timeout 900 python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/rl_pytest_rs1.log 2>&1; echo "pytest stack=1 rc=$?"; tail -1 gpurun_out/rl_pytest_rs1.log
cp /tmp/lib.orig paper_2508_08438_b200/libsafekv_b200.so
for w in 4 5 2; do timeout 600 python bench.py --workload $w --no-cpu-baseline > gpurun_out/rl_wl$w.json 2>/dev/null
python - gpurun_out/rl_wl$w.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "epoch avg", d["step_breakdown"]["epoch_ms"])
PY
done
