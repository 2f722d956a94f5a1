python -m pytest tests -m gpu -q -p no:cacheprovider -x -k "render or binning or mapping or dp or store or keyframe or loopclose or sample" > gpurun_out/t12.log 2>&1; tail -3 gpurun_out/t12.log
for v in main fwd0 old; do
  if [ $v = main ]; then V=""; else V=$v; fi
  SM_LIB_VARIANT=$V python bench.py --steps 300 --warmup 10 --no-cpu-baseline > gpurun_out/b12_$v.log 2>&1
  python -c "
import json,sys;d=json.loads(open(sys.argv[1]).read().strip().splitlines()[-1])
print(sys.argv[1], round(d['value'],1), round(d['e2e']['value'],1), round(d['ms_per_step'],4)); print({k:round(v['ms_per_step'],4) for k,v in d['stages'].items()})" gpurun_out/b12_$v.log
done
python tools/stream_bench.py --n 20000000 --length 1000 --keyframes 500 --modes resident,streamed > gpurun_out/r02_stream_c4full.json 2> gpurun_out/c4full.err; python -c "
import json;d=json.loads(open('gpurun_out/r02_stream_c4full.json').read().strip().splitlines()[-1]); print({k:(v['steps_per_s'] if isinstance(v,dict) else v) for k,v in d.items() if k in ('resident','streamed','overlap')})"
