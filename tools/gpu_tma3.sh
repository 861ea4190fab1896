#!/bin/bash
HB_TC_DEBUG=4 python tools/diag_tma1.py 512 64 32 64 3 1 1
timeout 600 python tools/diag_tma.py 2>&1 | sed -n 1,1p
python tools/diag_res.py | head -1
