# DRAM traffic per launch of each config's dominant kernel (roofline.traffic)
mkdir -p gpurun_out
M=dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum
timeout 900 ncu --metrics $M --clock-control none -k regex:batch_kernel -c 1 --csv python bench.py --config 3 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1_traffic_c3.csv 2> gpurun_out/traffic_c3.err; echo "c3 rc=$?"
timeout 900 ncu --metrics $M --clock-control none -k regex:cdist_kernel -c 1 --csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1_traffic_c4.csv 2> gpurun_out/traffic_c4.err; echo "c4 rc=$?"
timeout 900 ncu --metrics $M --clock-control none -k regex:long_kernel -c 2 --csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r1_traffic_c5.csv 2> gpurun_out/traffic_c5.err; echo "c5 rc=$?"
for c in 3 4 5; do grep -E "dram__|gpu__time" gpurun_out/r1_traffic_c$c.csv | awk -F'","' '{print $5" | "$(NF-2)" "$(NF-1)" "$NF}' | cut -c1-200; done
