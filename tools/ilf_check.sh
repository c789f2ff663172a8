#!/bin/bash
# Interleaved add/sub after a routing change: forced-route parity, the interleaved and
# fuzz GPU tests, then the graph-timed auto route against row-major.
python -m pytest tests/test_gpu_il_routes.py tests/test_gpu_addsub.py tests/test_gpu_fuzz.py -x -q > gpurun_out/ilf_tests.log 2>&1
python tools/il_graph.py --only 0,rows > gpurun_out/il_graph_auto.jsonl 2>&1
