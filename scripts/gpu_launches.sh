#!/bin/bash
# Launch list (ncu, per-kernel durations) of one QFT simulation at ${Q:-30} qubits.
mkdir -p gpurun_out
Q=${Q:-30}
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q$Q.csv python bench.py --qubits $Q --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_q$Q.csv ${THR:-1000} > gpurun_out/launches_q$Q.txt
tail -40 gpurun_out/launches_q$Q.txt
