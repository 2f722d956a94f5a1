#!/bin/bash
# Round-2 out-of-core runs: C4-lite (thrashing budget), full C4, C5 stress.
# Every mode runs --repeat times interleaved; each reports its median run.
python tools/stream_bench.py --budget 1100000 --modes resident,sync,streamed --repeat 3 > gpurun_out/r02_stream_c4lite.json 2> gpurun_out/c4lite.err
python -c "
import json;d=json.loads(open('gpurun_out/r02_stream_c4lite.json').read().strip().splitlines()[-1]); print('c4lite', {k: round(v['steps_per_s'],1) for k,v in d['runs'].items()}, d['overlap'], d['same_training'])"
if [ "$1" = "full" ]; then
python tools/stream_bench.py --n 20000000 --length 1000 --keyframes 500 --modes resident,streamed --repeat 3 > gpurun_out/r02_stream_c4full.json 2> gpurun_out/c4full.err
python -c "
import json;d=json.loads(open('gpurun_out/r02_stream_c4full.json').read().strip().splitlines()[-1]); print('c4full', {k: round(v['steps_per_s'],1) for k,v in d['runs'].items()}, d['overlap'], d['same_training'])"
fi
python tools/stress_bench.py --out gpurun_out/r02_stress_c5.json > gpurun_out/c5.out 2> gpurun_out/c5.err
python -c "
import json;d=json.loads(open('gpurun_out/r02_stress_c5.json').read()); print('c5', {k: round(v['steps_per_s'],1) for k,v in d['runs'].items()}, d['overlap'], d['vs_disk_floor'], d['cap_held'], d['disk'])"
