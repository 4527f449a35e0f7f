#!/bin/bash
mkdir -p gpurun_out
O=gpurun_out/ws_exp.txt
: > $O
NW_ITMA_WS=0 timeout 200 python tools/stream_exp.py c2k9 c2k5 c2k7 c3 >> $O 2>&1
timeout 200 python tools/stream_exp.py c2k9 c2k5 c2k7 c3 >> $O 2>&1
NW_STREAM=1 NW_STREAM_IT=80 timeout 200 python tools/stream_exp.py c2k9 c3 >> $O 2>&1
cat $O
