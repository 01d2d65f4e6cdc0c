#!/bin/bash
cd $GRAFT_REPO_ROOT
for e in "SKV_PF_GENERAL=1" "SKV_H16_PF_FRAC=6" "SKV_H16_PF_FRAC=8" "SKV_H16_PF_FRAC=4"; do
  env $e timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline > gpurun_out/abenv.json 2>/dev/null
  python3 -c "
import json; j=json.loads([l for l in open('gpurun_out/abenv.json') if l.startswith('{')][0])
print('$e', round(j['ms_per_step'],4), 'hs', round(j['roofline']['avg_launch_ms'],4), 'commit', j['step_breakdown']['commit_ms'], 'probe', j['step_breakdown']['chain_probe_ms'])"
done
