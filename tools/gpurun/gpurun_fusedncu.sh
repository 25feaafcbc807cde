#!/bin/bash
# ncu counters of kbg_grid_pass_dev at 56 atoms: the fused rho + H kernel (KBG_OPT_FUSED_PASS = 1) vs the
# two separate persistent kernels (0): duration, DMMA pipe, issue, warps, DRAM bytes, L2 hit rate
mkdir -p gpurun_out
M=gpu__time_duration.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct
for mode in 1 0; do
  for cfg in cubic56_200Ry super448_200Ry; do
  FUSED=$mode CFG=$cfg timeout 600 ncu --metrics $M --clock-control none --csv -k regex:'k_fused|k_persist' python -c "
import os, sys; sys.path.insert(0, '.')
import torch
from paper_1402_4247_b200 import _abi
from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4
f = Fe3O4.config(os.environ['CFG']); gp = GridPass(f.system); ix = gp.build_index()
gp.set_option(_abi.KBG_OPT_FUSED_PASS, int(os.environ['FUSED']))
dm = torch.from_numpy(f.dm(ix)).cuda(); v = torch.from_numpy(f.veff()).cuda()
rho = torch.empty((1, f.system.npts), dtype=torch.float64, device='cuda')
h = torch.empty((1, ix['nnz']), dtype=torch.float64, device='cuda')
gp.grid_pass_dev(dm, v, f.dV, rho, h); torch.cuda.synchronize()
" > gpurun_out/fusedncu_${mode}_$cfg.csv 2>&1
  echo "fused=$mode $cfg"; grep -E '"(k_fused|k_persist|.*k_fused|.*k_persist)' gpurun_out/fusedncu_${mode}_$cfg.csv | awk -F'","' '{print $5, $13, $15}' | sed 's/"//g' | sed 's/(anonymous namespace):://'
  done
done
