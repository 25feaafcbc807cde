for v in u1 u4 u8; do KBG_LIBKBGRID=$PWD/paper_1402_4247_b200/lib_var/$v/libkbgrid.so python tools/tridiag_grid_sweep.py 568,1040,2048 148 | sed "s/^/$v /"; done
KBG_LIBKBGRID=$PWD/paper_1402_4247_b200/lib_var/u4/libkbgrid.so python -m pytest tests/test_gpu_eigen.py -x -q 2>&1 | tail -1
