# round-2 DRAM traffic per launch of each config's dominant kernel, final kernels (roofline.traffic evidence)
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 600 ncu --metrics $M --clock-control none -k "regex:batch_kernel|seg_kernel" -c 4 --csv python bench.py --config 2 --steps 1 --warmup 3 --no-cpu-baseline --no-cdist > gpurun_out/r2_traffic_c2.csv 2> gpurun_out/traffic_c2.err; echo "c2 rc=$?"
timeout 900 ncu --metrics $M --clock-control none -k "regex:batch_kernel|seg_kernel" -c 4 --csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_traffic_c3.csv 2> gpurun_out/traffic_c3.err; echo "c3 rc=$?"
timeout 900 ncu --metrics $M --clock-control none -k regex:long_kernel -c 3 --csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r2_traffic_c5.csv 2> gpurun_out/traffic_c5.err; echo "c5 rc=$?"
for c in 2 3 5; do echo "== c$c"; grep -E "dram__|gpu__time" gpurun_out/r2_traffic_c$c.csv | awk -F'","' '{print substr($5,1,60)" | "$(NF-2)" "$(NF-1)" "$NF}'; done
