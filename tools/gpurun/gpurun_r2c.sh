#!/bin/bash
# round-2: GPU tests, kernel times (FP64 atomics and deterministic), short bench, ncu source profile of H
tag=${1:-r2c}; mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu_$tag.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$tag.log
timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 > gpurun_out/kernel_times_$tag.log 2>&1
timeout 300 python tools/kernel_times.py --schedules 3 --fallback 0 --det 1 --kernels h_accumulate >> gpurun_out/kernel_times_$tag.log 2>&1
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_$tag.json 2> gpurun_out/bench_$tag.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$tag.csv python -c "
import sys; sys.path.insert(0,'.')
from paper_1402_4247_b200.grid import GridPass
from paper_1402_4247_b200.system import Fe3O4
f=Fe3O4.config('cubic56_200Ry'); gp=GridPass(f.system); gp.build_index(); gp.build_index()
" > gpurun_out/ncu_setup_$tag.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_persist|k_phi_cache|k_build_tables" -c 6 -o gpurun_out/prof_$tag python bench.py --profile --no-e2e > gpurun_out/ncu_full_$tag.log 2>&1
echo "ncu rc=$?" >> gpurun_out/ncu_full_$tag.log
tail -n 3 gpurun_out/pytest_gpu_$tag.log; grep -o '"det": [01], "kernel": "[a-z_]*".*"median_ms": [0-9.]*' gpurun_out/kernel_times_$tag.log | sed 's/"plan".*"median/median/'; cut -c1-2500 gpurun_out/bench_$tag.json; tail -2 gpurun_out/ncu_full_$tag.log
