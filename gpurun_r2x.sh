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
