for x in 0 1; do for g in "" 1; do
echo "== xfirst=$x no_gather=$g"
KBG_NO_DM_GATHER=${g:-} KBG_XCHG_FIRST=$x timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29544 tools/e2e_probe.py ${1:-cubic56_200Ry} 2>&1 | grep -E "^\{|illegal|rror" | head -1 | cut -c1-300
done; done
