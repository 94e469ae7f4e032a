#!/bin/bash
# masked-path timing under experiment variants
export PYTHONPATH=.
python tools/time_mask.py
for v in ${VARIANTS:-4096}; do echo "variant $v"; DFSS_FLASH_VARIANT=$v python tools/time_mask.py; done
