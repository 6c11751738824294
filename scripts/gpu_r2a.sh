#!/bin/bash
# round 2 check: smoke, GPU parity tests, full bench line (incl. the stratified CPU baseline)
set -x
nproc; lscpu | grep "Model name"
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 1500 python -m pytest tests -m gpu -x -q --ignore=tests/test_headline_layout_gpu.py 2>&1 | tail -5
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_r2a.json 2> gpurun_out/bench_r2a.err; tail -3 gpurun_out/bench_r2a.err
cat gpurun_out/bench_r2a.json
