#!/bin/bash
# launch lists + one ncu --set full capture of a mid-run gate pass for the dense workloads at 28 qubits
mkdir -p gpurun_out
for W in "qaoa3reg --error-bound 1e-4" "random --layers 20"; do
  name=$(echo $W | cut -d' ' -f1)
  BQ="python bench.py --workload $W --qubits 28 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e --no-link"
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${name}28.csv $BQ > /dev/null 2>&1
  python scripts/launches.py gpurun_out/launches_${name}28.csv 1e18 > gpurun_out/launches_${name}28.txt
  tail -12 gpurun_out/launches_${name}28.txt
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_gate_pass_fast -s ${S:-40} -c 1 -o gpurun_out/prof_${name}28 -f $BQ > gpurun_out/ncu_${name}28.log 2>&1
  python scripts/ncu_summary.py gpurun_out/prof_${name}28.ncu-rep 25 2>&1 | tail -45
done
ls -la gpurun_out/*.ncu-rep
