#!/bin/bash
# Tests + stage profile + QAOA/QFT launch totals (iteration on the gate pass).
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -4 > gpurun_out/tests.txt
cat gpurun_out/tests.txt
timeout 600 python bench.py --workload qaoa3reg --qubits 30 --error-bound 1e-4 --steps 1 --warmup 1 --no-e2e 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('qaoa30', d['ms_per_step'], d['roofline']['phase_ms'], d['fidelity'])"
timeout 600 python bench.py --steps 1 --warmup 1 --no-e2e --no-cpu-baseline 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('qft34', d['ms_per_step'], d['roofline']['phase_ms'])"
