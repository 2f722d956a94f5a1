#!/bin/bash
# Round-2 closing evidence: the whole -m gpu suite, smoke(), the bench line
# (default and 300 steps), the C3 K = 8 line at G = 1, the reference arm.
set -u
python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02_smoke.log
python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench default rc=$?"
python bench.py --steps 300 --warmup 10 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 300 gpurun_out/r02_bench.json
python bench.py --steps 300 --warmup 10 --keyframes-per-step 8 > gpurun_out/r02_bench_c3_g1.json 2> gpurun_out/r02_bench_c3.err; echo "bench c3 rc=$?"
python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo "reference rc=$?"
tail -c 300 gpurun_out/r02_bench_reference.json
