N=$(python scripts/profile_solve.py 1 2 2>/dev/null | awk 'NR==1{a=$NF} NR==2{b=$NF} END{print b-a}')
echo "launches per solve: $N" > gpurun_out/warm_sum.log
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --launch-skip $N --launch-count $N --csv --log-file gpurun_out/c1_warm1.csv python scripts/profile_solve.py 1 2 > /dev/null 2>&1
timeout 120 python scripts/time_solve.py 1 20 >> gpurun_out/warm_sum.log 2>&1
