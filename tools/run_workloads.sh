#!/bin/bash
# Bench lines of every workload (SURVEY 8(d) configs 1, 3, 4, 5 and the system-prompt workload 6)
# beside the reference arm on the same config: gpurun_out/wl<N>.json, wl<N>_ref.json.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for w in ${WORKLOADS:-1 3 4 5 6}; do
  timeout 900 python bench.py --workload $w > gpurun_out/wl$w.json 2> gpurun_out/wl$w.err
  timeout 900 python bench.py --workload $w --impl reference --steps 3 --warmup 1 > gpurun_out/wl${w}_ref.json 2> gpurun_out/wl${w}_ref.err
  echo "workload $w rc done"
done
