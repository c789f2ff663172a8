mkdir -p gpurun_out
B="python bench.py --only C3,C4 --steps 3 --warmup 3"
$B > gpurun_out/mul_plain.json 2>&1; echo plain rc=$?; cat gpurun_out/mul_plain.json | tail -2
$B > /dev/null 2>&1 && ncu --set full --clock-control none --import-source on -k regex:k_mul_regs -s 2 -c 1 -o gpurun_out/prof_mul16 $B > gpurun_out/ncu_mul16.log 2>&1; echo ncu16 rc=$?
ncu --set full --clock-control none --import-source on -k regex:k_mul_smem -s 2 -c 1 -o gpurun_out/prof_mul64 $B > gpurun_out/ncu_mul64.log 2>&1; echo ncu64 rc=$?
