#!/bin/bash
export NW_ITMA_F32=1
timeout 300 python tools/prof_layer.py c2k9 > gpurun_out/prof_plain_r2l.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:input_transform_tma -s 1 -c 1 -o gpurun_out/prof_r2l_c2k9_itma32 python tools/prof_layer.py c2k9 > gpurun_out/ncu_r2l.log 2>&1
ncu -i gpurun_out/prof_r2l_c2k9_itma32.ncu-rep --page raw --csv > gpurun_out/prof_r2l_c2k9_itma32.raw.csv
ncu -i gpurun_out/prof_r2l_c2k9_itma32.ncu-rep --page source --csv > gpurun_out/prof_r2l_c2k9_itma32.source.csv
rm -f gpurun_out/prof_r2l_c2k9_itma32.ncu-rep
tail -2 gpurun_out/ncu_r2l.log
