#!/bin/bash
# round-2 iteration: GPU tests, kernel times (FP64 atomics / deterministic), A5 switch, setup launch list
tag=${1:-r2d}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 > gpurun_out/kernel_times_$tag.log 2>&1
timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 --det 1 --kernels h_accumulate >> gpurun_out/kernel_times_$tag.log 2>&1
timeout 600 python tools/a5_switch.py > gpurun_out/a5_$tag.jsonl 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/launches_setup_$tag.csv python -c "
import sys; sys.path.insert(0,'.')
from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4
f=Fe3O4.config('cubic56_200Ry'); gp=GridPass(f.system); gp.build_index(); gp.build_index()
" > gpurun_out/ncu_setup_$tag.log 2>&1
tail -n 3 gpurun_out/pytest_gpu_$tag.log; grep -o '"det": [01], "sparse": [0-9]*, "kernel": "[a-z_]*".*"median_ms": [0-9.]*' gpurun_out/kernel_times_$tag.log | sed 's/"plan".*"median/median/'; cut -c1-400 gpurun_out/a5_$tag.jsonl; grep -E "k_phi_cache|k_build_tables|k_cover_masks|k_tasks" gpurun_out/launches_setup_$tag.csv | cut -c1-250 | head
