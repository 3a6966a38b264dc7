# c5 per-launch times after the abort-check fix: 4 columns (default, R16 built), 4 columns without R16, 2 columns
cd paper_2404_05708_b200
for v in "" _lc4r8 _lc2; do
  for r in 0 8; do
  FFD_LONG_R=$r FFD_LIB=$PWD/libffd$v.so timeout 120 python ../scripts/c5_launches.py 3 l2 > ../gpurun_out/r2l_c5$v.r$r.json 2>&1; echo "lib$v R=$r rc=$?"; cut -c1-300 ../gpurun_out/r2l_c5$v.r$r.json
  done
done
