#!/bin/bash
# time every exp/<variant>/ library with tools/time_flash.py (c2, c3, c4 vs SDPA)
for d in ${VARIANTS:-$(ls exp)}; do
  echo "== $d"; DFSS_LIB=exp/$d/libdfss_sm100a.so timeout -s KILL 120 python tools/time_flash.py 2>&1 | tail -3
done
