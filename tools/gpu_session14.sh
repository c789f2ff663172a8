B="python bench.py --only C3,C4 --steps 3 --warmup 3 --no-e2e --no-cpu"
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_mul_smem -s 2 -c 1 -o gpurun_out/prof_mul64c $B > /dev/null 2>&1; echo rc=$?
