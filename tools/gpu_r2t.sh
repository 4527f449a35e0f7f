#!/bin/bash
# source-level ncu of the c2k9 input / output transforms; per-kernel breakdown of c4a / c4b / c5
TAG=r2t
mkdir -p gpurun_out
for L in c4a c4b c5_conv1 c5_deconv c3; do KERNELS=1 timeout 120 python tools/time_layers.py $L; done > gpurun_out/${TAG}_layers.txt 2>&1
timeout 120 python tools/prof_layer.py c2k9 > /dev/null 2>&1
for K in input_transform output_transform; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$K -s 1 -c 1 \
    -o gpurun_out/prof_${TAG}_c2k9_$K python tools/prof_layer.py c2k9 > gpurun_out/ncu_${TAG}_$K.log 2>&1; echo "ncu $K rc=$?"
done
for r in gpurun_out/prof_${TAG}_*.ncu-rep; do
  b=$(basename $r .ncu-rep)
  ncu -i $r --page raw --csv > gpurun_out/$b.raw.csv 2>/dev/null
  ncu -i $r --page source --csv > gpurun_out/$b.source.csv 2>/dev/null
  ncu -i $r --page details --csv > gpurun_out/$b.details.csv 2>/dev/null
done
cat gpurun_out/${TAG}_layers.txt
