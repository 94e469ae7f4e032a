#!/bin/bash
# run each selected GPU test in its own process with a hard timeout (hang triage)
SEL=${1-"flash or 16bit"}
for t in $(python -m pytest tests/test_gpu_parity.py -q --collect-only -k "$SEL" 2>/dev/null | grep "::"); do
  timeout -s KILL ${T:-45} python -m pytest -q -x "$t" > /tmp/one.log 2>&1
  rc=$?
  echo "rc=$rc $t"
  if [ $rc -ne 0 ]; then tail -5 /tmp/one.log; fi
done
