#!/bin/bash
# A/B of library variants in one gpurun call: parity subset, then the C2 bench per variant.
#   bash tools/ab_round2.sh "main pair q6"
VARIANTS=${1:-"main"}
python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "render or binning or mapping or dp" > gpurun_out/ab_tests.log 2>&1; tail -2 gpurun_out/ab_tests.log
for v in $VARIANTS; do
  if [ $v = main ]; then V=""; else V=$v; fi
  SM_LIB_VARIANT=$V python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "backward or edge_cases or full_size or optimization_step" > gpurun_out/ab_tests_$v.log 2>&1; echo "$v tests: $(tail -1 gpurun_out/ab_tests_$v.log)"
  SM_LIB_VARIANT=$V python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/ab_$v.log 2>&1
  python -c "
import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],4)); print({k:round(v['ms_per_step'],4) for k,v in d['stages'].items()})" gpurun_out/ab_$v.log
done
