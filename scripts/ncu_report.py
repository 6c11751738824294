"""One text summary of an ncu --set full report for profiles/: headline
metrics, stall reasons and the hottest CUDA lines."""
import subprocess
import sys

rep = sys.argv[1]
here = sys.path[0]
print("# ncu --set full --clock-control none (see profiles/README.md for the launch)")
for script, args in (("ncu_summary.py", []), ("ncu_stalls.py", [])):
    out = subprocess.run([sys.executable, f"{here}/{script}", rep] + args, capture_output=True, text=True).stdout
    sys.stdout.write(out)
print("# hottest CUDA lines (share of executed instructions / of stall samples)")
out = subprocess.run([sys.executable, f"{here}/ncu_srcmap.py", rep, "15"], capture_output=True, text=True).stdout
sys.stdout.write(out)
