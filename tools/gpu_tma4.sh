#!/bin/bash
echo default; timeout 600 python tools/diag_tma.py 2>&1 | sed -n 1,1p
echo P2D; HB_TMA_P2D=1 timeout 600 python tools/diag_tma.py 2>&1 | sed -n 1,1p
