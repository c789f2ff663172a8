set -x
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo smoke rc=$?
python -m pytest tests -m gpu -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
B="python bench.py --steps 2 --warmup 3 --no-secondary --no-e2e --no-cpu"
$B > gpurun_out/ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file gpurun_out/launches.csv $B > gpurun_out/ncu1.log 2>&1; echo ncu1 rc=$?
$B > gpurun_out/ncu_plain2.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:k_addsub_team -s 8 -c 4 -o gpurun_out/prof_addsub $B > gpurun_out/ncu2.log 2>&1; echo ncu2 rc=$?
