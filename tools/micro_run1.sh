cd tools/micro
for w in 6 8 16 32 64; do for pf in 0 1; do for mb in 4 5 6; do for sys in 1 0; do
  r=$(./p2p_bench_s_w${w}_pf${pf}_b$mb 24 10 0 $sys | grep '^{')
  echo "w=$w pf=$pf minb=$mb $r"
done; done; done; done
