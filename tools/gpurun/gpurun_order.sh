mkdir -p gpurun_out; : > gpurun_out/plan.log
for c in ${CONFIGS:-cubic56_200Ry sweep56_100Ry sweep56_150Ry super448_200Ry}; do
timeout 300 python tools/kernel_times.py --config $c --schedules 3 --fallback 0 >> gpurun_out/plan.log 2>&1
done
cat gpurun_out/plan.log
