#!/bin/bash
# One `ncu --set full` capture of the top stencil launch per config, exported
# to raw CSV under gpurun_out/prof/ (profiles/summarize_ncu.py reads them).
#   tools/ncu_full.sh "vec_c2:c2 vec_c3o8:c3o8 vecq_c3o16:c3o16"
set -u
mkdir -p gpurun_out/prof
for item in $1; do
  name=${item%%:*}; cfg=${item##*:}
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:${KREGEX:-acoustic3d} -s 10 -c 1 \
    -f -o gpurun_out/prof/$name python bench.py --config $cfg --steps 1 --warmup 1 --no-cpu-baseline \
    > gpurun_out/prof/$name.log 2>&1
  ncu -i gpurun_out/prof/$name.ncu-rep --page raw --csv > gpurun_out/prof/$name.raw.csv 2>/dev/null
  ncu -i gpurun_out/prof/$name.ncu-rep --page details --csv > gpurun_out/prof/$name.details.csv 2>/dev/null
  ncu -i gpurun_out/prof/$name.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/$name.sass.csv 2>/dev/null
  ls -la gpurun_out/prof/$name.ncu-rep; rm -f gpurun_out/prof/$name.ncu-rep
  echo "$name done"
done
