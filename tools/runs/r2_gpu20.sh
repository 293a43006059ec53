#!/bin/bash
# A/B across two library builds (A = before, B = after: queue shift of the
# radius <= 6 form on the ALU pipe), alternating processes
mkdir -p gpurun_out/r2t
L=paper_1609_03361_b200
for k in 1 2 3; do
  for v in A B; do
    cp $L/libsf_b200_$v.so $L/libsf_b200.so
    timeout 600 python tools/ab_time.py c3o12 6 "" | sed "s/\"variant\": \"\"/\"variant\": \"$v\"/" >> gpurun_out/r2t/ab_c3o12.jsonl 2>&1
  done
done
cp $L/libsf_b200_B.so $L/libsf_b200.so
