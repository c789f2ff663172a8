python -m pytest tests/test_gpu_long.py tests/test_gpu_host_api.py -q -x 2>&1 | tail -2
python bench.py --only C5 --steps 5 --warmup 2 2>&1 | tail -c 500
