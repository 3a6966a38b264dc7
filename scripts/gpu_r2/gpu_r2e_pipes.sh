# two-column c2 cell vs one-column; ncu of FMNMX alone (which pipe)
cd tools/microbench
./pipes cell_xsq > ../../gpurun_out/r2_pipes_cell2.jsonl 2>&1; echo "rc=$?"
./pipes FMNMX > /dev/null 2>&1 && ncu --set full --clock-control none -k regex:op_kernel -c 6 -o ../../gpurun_out/r2_fmnmx_ncu ./pipes FMNMX > ../../gpurun_out/r2_fmnmx_ncu.log 2>&1; echo "ncu rc=$?"
