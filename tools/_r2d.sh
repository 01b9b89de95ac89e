timeout 120 ./tools/launch_floor > gpurun_out/launch_floor.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/compress_launches2.csv env GEN=1 STEPS=2 python tools/profile_step.py > /dev/null 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2d.log 2>&1; echo "rc $?" >> gpurun_out/gputest_r2d.log
