#!/bin/bash
mkdir -p gpurun_out
for shp in "l1 512 64 32 64 3 1 1" "l3 512 256 8 256 3 1 1"; do set -- $shp; name=$1; shift
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_conv_tma -s 2 -c 1 -o gpurun_out/prof_convpair_$name python tools/diag_conv_pair.py "$@" > /dev/null 2>&1; echo "ncu $name rc=$?"
  ncu -i gpurun_out/prof_convpair_$name.ncu-rep --page raw --csv > gpurun_out/ncu_raw_convpair_${name}_r02.csv 2>/dev/null
  rm -f gpurun_out/prof_convpair_$name.ncu-rep
done
