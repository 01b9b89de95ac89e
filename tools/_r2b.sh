timeout 120 ./tools/launch_floor > gpurun_out/launch_floor.txt 2>&1
timeout 300 python tools/step_breakdown.py > gpurun_out/step_breakdown.txt 2>&1
