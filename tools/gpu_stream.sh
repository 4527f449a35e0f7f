#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/stream_exp2.txt
: > $O
timeout 120 python tools/stream_exp.py c2k9 c2k5 >> $O 2>&1
for ot in 36 48 64; do
  NW_STREAM=2 NW_STREAM_OT=$ot timeout 120 python tools/stream_exp.py c2k9 c2k5 >> $O 2>&1
done
for cfg in "56 40" "64 40" "72 36" "80 30"; do set -- $cfg
  NW_STREAM=3 NW_STREAM_IT=$1 NW_STREAM_OT=$2 timeout 120 python tools/stream_exp.py c2k9 c2k5 >> $O 2>&1
done
cat $O
