for h in 0 1; do DOTG_K16_HYBRID=$h python tools/c3_probe.py; done > gpurun_out/c3_ab.jsonl 2>&1
echo rc=$?
DOTG_K16_HYBRID=0 python -m pytest tests -m gpu -x -q -k "test_gpu_mul and (m16 or 16 or config)" > gpurun_out/pt_c3_old.log 2>&1; echo rc_old=$?
python -m pytest tests -m gpu -x -q -k "test_gpu_mul or acceptance or fuzz or kara" > gpurun_out/pt_c3.log 2>&1; echo rc_new=$?
tail -1 gpurun_out/pt_c3_old.log; tail -1 gpurun_out/pt_c3.log
