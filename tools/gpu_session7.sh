B="python bench.py --only C5 --steps 3 --warmup 2"
$B > gpurun_out/c5_plain.json 2>&1; echo rc=$?; tail -c 600 gpurun_out/c5_plain.json
$B > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_long -c 30 --csv --log-file gpurun_out/c5_launches.csv $B > /dev/null 2>&1; echo ncu rc=$?
