#!/bin/bash
timeout 600 python tools/diag_tma.py 2>&1 | tail -12
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_limbs_nhwc -c 2 python tools/diag_tma1.py 512 64 32 64 3 1 1 2>&1 | grep -E "duration|bytes" | head -6
