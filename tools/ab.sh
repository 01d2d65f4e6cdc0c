#!/bin/bash
# A/B timing of library variants built with `make variant V=<name> VFLAGS=...`:
#   tools/ab.sh <name>[:bench flags]...   -> gpurun_out/ab_<name>.json (bench line per variant)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
# variants/ is gpurun-ignored: run A/B variants by removing that line from .gpurunignore for the call
cp paper_2508_08438_b200/libsafekv_b200.so /tmp/libsafekv_b200.so.orig
for spec in "$@"; do
  v="${spec%%:*}"; flags=""; [ "$spec" != "$v" ] && flags="${spec#*:}"
  tag="$v$(echo "$flags" | tr -d ' -')"
  cp "variants/$v/libsafekv_b200.so" paper_2508_08438_b200/libsafekv_b200.so
  timeout 600 python bench.py --steps 8 --warmup 3 --no-cpu-baseline $flags > "gpurun_out/ab_$tag.json" 2> "gpurun_out/ab_$tag.err"
  python3 -c "
import json,sys; j=json.loads([l for l in open('gpurun_out/ab_$tag.json') if l.startswith('{')][0])
print('$tag', round(j['ms_per_step'],4), 'hs', round(j['roofline']['avg_launch_ms'],4), 'commit', j['step_breakdown']['commit_ms'], 'probe', j['step_breakdown']['chain_probe_ms'])"
done
cp /tmp/libsafekv_b200.so.orig paper_2508_08438_b200/libsafekv_b200.so
