#!/bin/bash
# ncu --set full (with source): c2k9 contraction after the epilogue fix; C4a / C4b input transforms
TAG=r2x
mkdir -p gpurun_out
for spec in "c2k9 contraction" "c4a input_transform" "c4b input_transform"; do set -- $spec
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
