# ncu of the c5 long kernel: 4 columns (no R16) and 2 columns, after the abort-check fix
cd paper_2404_05708_b200
CMD="python ../scripts/c5_launches.py 1 l2"
for v in _lc4r8 _lc2; do
FFD_LIB=$PWD/libffd$v.so timeout 120 $CMD > /dev/null 2>&1 && \
FFD_LIB=$PWD/libffd$v.so timeout 900 ncu --set full --clock-control none --import-source on -k regex:long_kernel -s 1 -c 1 -o ../gpurun_out/r2m_c5$v $CMD > ../gpurun_out/r2m_ncu$v.log 2>&1; echo "ncu $v rc=$?"
done
