cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2 3; do timeout 300 python bench.py --no-cpu-baseline > gpurun_out/x_$i.json 2>/dev/null
python - gpurun_out/x_$i.json <<'PY'
import json,sys
d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d["value"]/1e9,4), round(d["ms_per_step"],4), "e2e", round(d["e2e"]["value"]/1e9,4), d["stage_ms_last"], d["step_breakdown"]["commit_ms"])
PY
done
SKV_H16_PF_WARPS=8 timeout 300 python bench.py --no-cpu-baseline > gpurun_out/x_env.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/x_env.json').read().strip().splitlines()[-1]); print('env', d['ms_per_step'])"
timeout 300 python bench.py > gpurun_out/x_full.json 2>/dev/null; python -c "
import json; d=json.loads(open('gpurun_out/x_full.json').read().strip().splitlines()[-1]); print('full', d['ms_per_step'], d['e2e']['value'])"
T="tests/test_gpu_graphs.py tests/test_gpu_golden.py::test_config1_golden tests/test_gpu_parity.py::test_parity_b16_w32 tests/test_gpu_prefetch.py::test_step_host_pipeline_parity"
for tool in memcheck racecheck synccheck initcheck; do
  extra=""; [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1200 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 30 python -m pytest $T -x -q -p no:cacheprovider > gpurun_out/x_san_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/x_san_$tool.log | tail -2 | tr '\n' ' ')"
done
