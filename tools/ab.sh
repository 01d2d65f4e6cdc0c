#!/bin/bash
# A/B timing of library variants built with `make variant V=<name> VFLAGS=...`:
#   tools/ab.sh <name>...   -> gpurun_out/ab_<name>.json (bench line per variant)
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_2508_08438_b200/libsafekv_b200.so /tmp/libsafekv_b200.so.orig
for v in "$@"; do
  cp "variants/$v/libsafekv_b200.so" paper_2508_08438_b200/libsafekv_b200.so
  timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > "gpurun_out/ab_$v.json" 2> "gpurun_out/ab_$v.err"
done
cp /tmp/libsafekv_b200.so.orig paper_2508_08438_b200/libsafekv_b200.so
