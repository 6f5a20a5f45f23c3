for g in 16 8 4; do echo "G=$g"; DIFFMPC_GROUP=$g python tools/quick_bench.py 2>&1 | head -5; done
DIFFMPC_GROUP=8 python tools/parity_report.py 2>&1 | grep -v Warn | awk '{print $1,$2,$3,$5,$7,$9,$11,$13,$15,$17,$19,$22,$24}' | grep -v "^J" > gpurun_out/parity_g8.txt
DIFFMPC_GROUP=4 python tools/parity_report.py 2>&1 | grep -v Warn | awk '{print $1,$2,$3,$5,$7,$9,$11,$13,$15,$17,$19,$22,$24}' | grep -v "^J" > gpurun_out/parity_g4.txt
awk '$5>0 || $10>0' gpurun_out/parity_g8.txt gpurun_out/parity_g4.txt
