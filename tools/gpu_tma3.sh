#!/bin/bash
HB_TC_DEBUG=4 python tools/diag_tma1.py 512 64 32 64 3 1 1
echo "default (P2D for n=64, P2/128 for n>=128)"; timeout 600 python tools/diag_tma.py 2>&1 | sed -n 1,13p
echo "HB_TMA_NT=64 (P2D everywhere)"; HB_TMA_NT=64 timeout 600 python tools/diag_tma.py 2>&1 | sed -n 1,6p
echo "P1 for n=64"; HB_TMA_P1=1 timeout 600 python tools/diag_tma.py 2>&1 | sed -n 1,1p
