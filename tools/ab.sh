#!/bin/bash
# A/B timing of exp/<variant> libraries on one box, interleaved (REPS rounds); CONFIGS / DFSS_MODE as in time_flash.py
for r in $(seq ${REPS:-3}); do
  for d in "$@"; do
    echo "== $d"; DFSS_LIB=exp/$d/libdfss_sm100a.so timeout -s KILL 120 python tools/time_flash.py 2>&1 | tail -3
  done
done
