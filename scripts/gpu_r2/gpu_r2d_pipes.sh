# microbenchmarks: the new c2-cell chain variants + ncu --set full of the cell mixes (roofline denominator)
cd tools/microbench
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm --format=csv
./pipes > ../../gpurun_out/r2_pipes.jsonl 2>&1; echo "pipes rc=$?"
./pipes mixcells_ > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:mix_kernel -c 4 -o ../../gpurun_out/r2_mix_ncu ./pipes mixcells_ > ../../gpurun_out/r2_mix_ncu.log 2>&1; echo "ncu mix rc=$?"
./pipes cell_xsq_fmnmx3_R12_shfl1_w16 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cell_kernel -c 2 -o ../../gpurun_out/r2_cell_fmnmx3_ncu ./pipes cell_xsq_fmnmx3_R12_shfl1_w16 > ../../gpurun_out/r2_cell_ncu.log 2>&1; echo "ncu cell rc=$?"
./pipes cell_xsq_split_int_R12_shfl1_w16 > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:cell_kernel -c 2 -o ../../gpurun_out/r2_cell_split_ncu ./pipes cell_xsq_split_int_R12_shfl1_w16 >> ../../gpurun_out/r2_cell_ncu.log 2>&1; echo "ncu cell2 rc=$?"
