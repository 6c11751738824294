#!/bin/bash
# Launch list of one simulation of workload W at Q qubits (extra bench args in A).
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$W$Q.csv python bench.py --workload $W --qubits $Q --steps 1 --warmup 0 --no-cpu-baseline --no-e2e $A > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_$W$Q.csv ${THR:-1e18} > gpurun_out/launches_$W$Q.txt
tail -25 gpurun_out/launches_$W$Q.txt
