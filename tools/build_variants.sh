#!/bin/bash
# Builds libkbgrid.so variants for timing experiments:
#   tools/build_variants.sh NAME "-DFOO=1 -DBAR=2" [NAME2 "FLAGS2" ...]
# -> paper_1402_4247_b200/lib_var/NAME/libkbgrid.so (load with KBG_LIBKBGRID=...)
set -e
cd "$(dirname "$0")/../paper_1402_4247_b200/csrc"
while [ $# -ge 2 ]; do
  make -j8 OUT=../lib_var/$1 EXTRA="$2" ../lib_var/$1/libkbgrid.so > /dev/null
  grep -h -A3 "k_persist" ../lib_var/$1/obj/kb_persist.ptxas.log | grep -E "Used|spill" | sed "s/^/$1: /"
  shift 2
done
