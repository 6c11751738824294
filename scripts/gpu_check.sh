#!/bin/bash
# Quick HEAD check: GPU parity suite, smoke, headline bench line.
mkdir -p gpurun_out
B=gpurun_out; T=${T:-chk}
timeout 1800 python -m pytest tests -m gpu -q -x 2>&1 | tail -15 > $B/${T}_tests.txt; tail -3 $B/${T}_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $B/${T}_smoke.txt 2>&1; tail -1 $B/${T}_smoke.txt
timeout 1200 python bench.py > $B/${T}_bench_qft34.json 2> $B/${T}_bench_qft34.err; tail -c 600 $B/${T}_bench_qft34.json
