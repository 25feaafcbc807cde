mkdir -p gpurun_out
timeout 300 python bench.py --profile --no-e2e --config super448_200Ry > gpurun_out/plain448.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_persist" -c 2 -o gpurun_out/prof448_r06 python bench.py --profile --no-e2e --config super448_200Ry > gpurun_out/ncu448.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu448.log
