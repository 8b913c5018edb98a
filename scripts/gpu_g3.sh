timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/g3_tests.log 2>&1
timeout 120 python scripts/time_solve.py 1 30 > gpurun_out/g3_time.log 2>&1
timeout 120 python scripts/time_solve.py 4 5 >> gpurun_out/g3_time.log 2>&1
N=$(python scripts/profile_solve.py 1 2 2>/dev/null | awk 'NR==1{a=$NF} NR==2{b=$NF} END{print b-a}')
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --launch-skip $N --launch-count $N --csv --log-file gpurun_out/g3_launches.csv python scripts/profile_solve.py 1 2 > /dev/null 2>&1
