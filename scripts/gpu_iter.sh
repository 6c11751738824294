#!/bin/bash
# Iteration session: GPU tests (optionally filtered), then the QFT-34 stage profile.
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x ${TESTS:-} 2>&1 | tail -15 > gpurun_out/tests.txt
cat gpurun_out/tests.txt
timeout 300 python scripts/stage_profile.py qft 34 20 2 > gpurun_out/stages_qft34.txt 2>&1
head -12 gpurun_out/stages_qft34.txt | cut -c1-400
