n=${1:-2}; tag=${2:-x}; mkdir -p gpurun_out; out=gpurun_out/p2p_n${n}_$tag.log; : > $out
timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -n 2 >> $out
port=29600
for c in cubic56_200Ry super448_200Ry super1512_200Ry; do
  port=$((port+1))
  timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $n --master-addr 127.0.0.1 --master-port $port tools/p2p_check.py $c 2>&1 | grep '^{' >> $out
done
cat $out
