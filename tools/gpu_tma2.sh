#!/bin/bash
for d in 0 1; do echo "dbg=$d"; HB_TC_DEBUG=$d timeout 600 python tools/diag_tma.py 2>&1 | sed -n 1,13p; done
