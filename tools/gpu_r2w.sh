#!/bin/bash
# ncu --set full (with source) of fused_c1 (C5 conv1), fused_co (C5 deconv), C4b's input transform
TAG=r2w
mkdir -p gpurun_out
for spec in "c5_conv1 fused_c1" "c5_deconv fused_co_kernel" "c4b input_transform" "c4a output_transform"; do set -- $spec
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
ls gpurun_out | grep $TAG
