#!/bin/bash
# L2-residency experiment: the chunk pipeline (NW_PIPE_CHUNKS) at chunk counts small enough that
# one chunk's V and M' stay in the 126 MB L2
for k in 1 8 16 32; do
  echo "== NW_PIPE_CHUNKS=$k"
  NW_PIPE_CHUNKS=$k KERNELS=1 timeout 300 python tools/time_layers.py c2k9 c2k5 2>&1 | tail -5
done
