for v in "XSMS=8" "XSMS=8 KBG_NO_DM_GATHER=1" "XSMS=8 KBG_NO_ZERO_COPY=1 KBG_NO_ZERO_COPY_OUT=1" "XSMS=8 KBG_NO_DM_GATHER=1 KBG_NO_ZERO_COPY=1 KBG_NO_ZERO_COPY_OUT=1" "XSMS=8 PIN=0" "XSMS=16" "XSMS=8 KBG_XCHG_FIRST=0"; do
  env $v KBG_PHASE_TIMING=1 timeout 120 python tools/two_rank_probe.py 2>&1 | grep -E "errors|phases" | cut -c1-330
done
