#!/bin/bash
# Fixed-state A/B of library builds (tools/kernel_ab.py), interleaved:
#   bash tools/kernel_ab.sh "main direct main direct"
for v in ${1:-main}; do
  if [ $v = main ]; then V=""; else V=$v; fi
  SM_LIB_VARIANT=$V python tools/kernel_ab.py --reps ${REPS:-10} 2>/dev/null | tail -1
done
