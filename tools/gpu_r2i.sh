#!/bin/bash
python -m pytest tests/test_gpu_depthwise.py -q -p no:cacheprovider -x -k "shape3" 2>&1 | grep -E "\[nw\]|passed|failed" | head
NW_DEBUG_SYNC=1 python -m pytest tests/test_gpu_depthwise.py -q -p no:cacheprovider 2>&1 | grep -E "\[nw\]|passed|failed" | head
python -m pytest tests/test_gpu_depthwise.py -q -p no:cacheprovider 2>&1 | grep -E "\[nw\]|passed|failed" | head
