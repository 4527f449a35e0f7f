#!/bin/bash
# ncu --set full (with source page) of chosen kernels: bash tools/gpu_ncu.sh <tag> "<layer> <kernel regex>" ...
# default: the c2k9 contraction and the C4a / C4b input transforms (round-2 capture r2x)
TAG=${1:-r2x}
shift
SPECS=("$@")
[ ${#SPECS[@]} -eq 0 ] && SPECS=("c2k9 contraction" "c4a input_transform" "c4b input_transform")
mkdir -p gpurun_out
for spec in "${SPECS[@]}"; do set -- $spec
  timeout 120 python tools/prof_layer.py $1 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$2 -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_$1_$2 python tools/prof_layer.py $1 > gpurun_out/ncu_${TAG}_$1.log 2>&1; echo "ncu $1 $2 rc=$?"
done
for r in gpurun_out/prof_${TAG}_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page raw --csv > gpurun_out/$b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv > gpurun_out/$b.source.csv 2>/dev/null
  rm -f $r
done
