#!/bin/bash
# 8-byte record lean variants (13/14) vs the 16-byte default (10/9): the
# sampler test file, then 30-iteration layout kernel time at C3 and C2.
# usage: bash tools/r2_rec8_ab.sh OUTDIR
out=${1:-gpurun_out/rec8_ab}
mkdir -p "$out"
timeout 900 python -m pytest tests/test_gpu_samplers.py -m gpu -x -q > "$out/tests.log" 2>&1
echo "tests rc=$?" >> "$out/tests.log"
for v in 10 13 10 13; do
    timeout 400 python tools/ab_speed.py c3 2 3 $v >> "$out/ab_c3.jsonl" 2>> "$out/ab.err"
done
for v in 10 13 9 14; do
    timeout 300 python tools/ab_speed.py c2 3 3 $v >> "$out/ab_c2.jsonl" 2>> "$out/ab.err"
done
