mkdir -p gpurun_out
timeout 300 python scripts/stage_profile.py qft 34 20 2 > gpurun_out/stages_qft34.txt 2>&1
timeout 300 python scripts/stage_profile.py qft 34 20 6 > gpurun_out/stages_qft34_i6.txt 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_q30.csv python bench.py --qubits 30 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
python scripts/launches.py gpurun_out/launches_q30.csv 1000 > gpurun_out/launches_q30.txt
