# c5 per-launch times: 4 columns (R=16 built / not built) vs 2 columns, all with the conflict-free ring
cd paper_2404_05708_b200
for v in "" _lc4r8 _lc2; do
  FFD_LIB=$PWD/libffd$v.so timeout 120 python ../scripts/c5_launches.py 3 l2 > ../gpurun_out/r2k_c5$v.json 2>&1; echo "lib$v rc=$?"; cat ../gpurun_out/r2k_c5$v.json | cut -c1-400
done
cd ..
CMD="python scripts/c5_launches.py 1 l2"
FFD_LIB=$PWD/paper_2404_05708_b200/libffd_lc2.so timeout 120 $CMD > /dev/null 2>&1 && \
FFD_LIB=$PWD/paper_2404_05708_b200/libffd_lc2.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:long_kernel -s 1 -c 1 -o gpurun_out/r2k_c5_lc2 $CMD > gpurun_out/r2k_ncu.log 2>&1; echo "ncu lc2 rc=$?"
FFD_LIB=$PWD/paper_2404_05708_b200/libffd_lc4r8.so timeout 120 $CMD > /dev/null 2>&1 && \
FFD_LIB=$PWD/paper_2404_05708_b200/libffd_lc4r8.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:long_kernel -s 1 -c 1 -o gpurun_out/r2k_c5_lc4r8 $CMD >> gpurun_out/r2k_ncu.log 2>&1; echo "ncu lc4r8 rc=$?"
