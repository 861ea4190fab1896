#!/bin/bash
for v in 2 4; do echo "shpf=$v"; HB_LIB_PATH=$PWD/paper_2309_04875_b200/lib/libhbrelu_shpf$v.so HB_TC_DEBUG=4 timeout 300 python tools/diag_conv_bounds.py 2>/dev/null | python -c "
import json,sys;d=json.load(sys.stdin)
for k,v in d.items():
    if k!='dbg': print(' ',k, round(v['ms'],4), v['stamps_clk']['wait_tmem_empty'], v['stamps_clk']['epi_tmem_read'])"; done
