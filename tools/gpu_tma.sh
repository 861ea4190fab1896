#!/bin/bash
timeout 600 python tools/diag_tma.py 2>&1 | tail -20
HB_TC_DEBUG=1 timeout 300 python tools/diag_tma.py 2>&1 | tail -12
