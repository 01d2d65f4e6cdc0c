#!/bin/bash
# A/B of k_hash_scan16 variants (make variant V=<name> VFLAGS=...): tools/hs_probe.py per variant
set -u
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
cp paper_2508_08438_b200/libsafekv_b200.so /tmp/libsafekv_b200.so.orig
for v in "$@"; do
  cp "variants/$v/libsafekv_b200.so" paper_2508_08438_b200/libsafekv_b200.so
  timeout 300 python tools/hs_probe.py > "gpurun_out/abhs_$v.log" 2>&1
  echo "$v $(grep median gpurun_out/abhs_$v.log)"
done
cp /tmp/libsafekv_b200.so.orig paper_2508_08438_b200/libsafekv_b200.so
