mkdir -p gpurun_out; out=gpurun_out/nvls_r11.log; : > $out
run() { python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $1 tools/p2p_check.py $2; }
NCCL_DEBUG=INFO timeout 600 bash -c "$(declare -f run); run 29701 super448_200Ry" > gpurun_out/nvls_info.log 2>&1
grep -iE "NVLS|nvls" gpurun_out/nvls_info.log | head -20 >> $out
echo "--- default" >> $out; grep '^{' gpurun_out/nvls_info.log >> $out
for a in Ring NVLS; do echo "--- NCCL_ALGO=$a" >> $out; NCCL_ALGO=$a timeout 600 bash -c "$(declare -f run); run $((29710 + RANDOM % 100)) super448_200Ry" 2>&1 | grep -E '^\{|rror' | head -3 >> $out; done
cat $out | cut -c1-400
