#!/bin/bash
# time tools/time_flash.py under DFSS_FLASH_VARIANT values (bring-up experiments)
for v in ${VARIANTS:-0 1 2 3 4 7}; do echo "variant $v"; DFSS_FLASH_VARIANT=$v timeout 120 python tools/time_flash.py; done
