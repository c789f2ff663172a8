B="python bench.py --steps 3 --warmup 3 --no-secondary --no-e2e --no-cpu"
$B > gpurun_out/plain10.log 2>&1; echo plain rc=$?
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:k_addsub -c 40 --csv --log-file gpurun_out/r01_launches_grouped.csv $B > /dev/null 2>&1; echo ncu1 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_addsub_grouped -s 3 -c 1 -o gpurun_out/prof_grouped $B > /dev/null 2>&1; echo ncu2 rc=$?
