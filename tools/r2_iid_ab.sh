#!/bin/bash
# i.i.d. kernel pipeline-depth A/B on the GPU box (round 2): correctness of
# the new variants, then layout kernel time at C5 / C3 / C2 per variant.
# usage: bash tools/r2_iid_ab.sh OUTDIR
out=${1:-gpurun_out/iid_ab}
mkdir -p "$out"
timeout 900 python -m pytest tests/test_gpu_samplers.py tests/test_gpu_parity.py -m gpu -x -q \
    -k "iid or batches_count or accounting or cooling_fractions or switch_point" > "$out/tests.log" 2>&1
echo "tests rc=$?" >> "$out/tests.log"
for v in 8 2 4 6 7 1 3 5; do
    timeout 300 python tools/ab_speed.py c5 2 3 $v '{"sampling": 1}' >> "$out/ab_c5.jsonl" 2>> "$out/ab.err"
done
for v in 8 4 7 2 6; do
    timeout 400 python tools/ab_speed.py c3 2 3 $v '{"sampling": 1}' >> "$out/ab_c3.jsonl" 2>> "$out/ab.err"
done
for v in 8 4 7; do
    timeout 300 python tools/ab_speed.py c2 2 3 $v '{"sampling": 1}' >> "$out/ab_c2.jsonl" 2>> "$out/ab.err"
done
