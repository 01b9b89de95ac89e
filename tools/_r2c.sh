timeout 120 ./tools/launch_floor > gpurun_out/launch_floor.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/compress_launches.csv env GEN=1 STEPS=2 python tools/profile_step.py > /dev/null 2>&1
timeout 300 ncu --set full --import-source on --clock-control none -k regex:select_kernel -s 1 -c 1 -o gpurun_out/k3_r2 env GEN=1 STEPS=1 python tools/profile_step.py > /dev/null 2>&1
ls gpurun_out
