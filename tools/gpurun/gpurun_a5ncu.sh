#!/bin/bash
# ncu counters of the H kernel with every task on DMMA (threshold 0) and every task on the point-exact
# DFMA path (threshold 255): duration, FP64 / DMMA pipe utilisation, issue, shared-memory wavefronts
M=gpu__time_duration.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active
for thr in 0 255; do
  A5_THR=$thr ncu --metrics $M --clock-control none --csv -k regex:k_persist python -c "
import os, sys; sys.path.insert(0, '.')
import torch
from paper_1402_4247_b200 import _abi
from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4
f = Fe3O4.config('cubic56_200Ry'); gp = GridPass(f.system); ix = gp.build_index()
gp.set_option(_abi.KBG_OPT_SPARSE_DFMA, int(os.environ['A5_THR']))
v = torch.from_numpy(f.veff()).cuda(); h = torch.empty((1, ix['nnz']), dtype=torch.float64, device='cuda')
gp.hamiltonian_accumulate_dev(v, f.dV, h); torch.cuda.synchronize()
" > gpurun_out/a5ncu_$thr.csv 2>&1
  echo "threshold $thr"; grep k_persist gpurun_out/a5ncu_$thr.csv | awk -F'","' '{print $13, $15}' | sed 's/"//g'
done
