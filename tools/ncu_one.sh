#!/bin/bash
# One `ncu --set full` capture: tools/ncu_one.sh NAME CONFIG KERNEL_REGEX [SKIP]
# (demangled names, so the regex can pin template arguments), exported to raw /
# details / SASS-source CSV under gpurun_out/prof/.
set -u
name=$1; cfg=$2; kre=$3; skip=${4:-10}
mkdir -p gpurun_out/prof
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base demangled \
  -k "regex:$kre" -s $skip -c 1 -f -o gpurun_out/prof/$name \
  python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline > gpurun_out/prof/$name.log 2>&1
ncu -i gpurun_out/prof/$name.ncu-rep --page raw --csv > gpurun_out/prof/$name.raw.csv 2>/dev/null
ncu -i gpurun_out/prof/$name.ncu-rep --page details --csv > gpurun_out/prof/$name.details.csv 2>/dev/null
ncu -i gpurun_out/prof/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/$name.sass.csv 2>/dev/null
ls -la gpurun_out/prof/$name.ncu-rep; rm -f gpurun_out/prof/$name.ncu-rep
echo "$name done"
