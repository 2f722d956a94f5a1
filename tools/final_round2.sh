#!/bin/bash
# Round-2 closing evidence: the whole -m gpu suite, smoke(), the bench line
# (default and 300 steps), the C3 K = 8 line at G = 1, the reference arm, then
# the ncu launch list and one --set full capture of a mapping step (each ncu
# pass only after the plain bench exited 0).
set -u
python -m pytest tests -m gpu -q > gpurun_out/r02_gpu_tests.log 2>&1; echo "gpu tests rc=$?"; tail -2 gpurun_out/r02_gpu_tests.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02_smoke.log
python bench.py > gpurun_out/r02_bench_default.json 2> gpurun_out/r02_bench_default.err; echo "bench default rc=$?"
python bench.py --steps 300 --warmup 10 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; rc=$?; echo "bench rc=$rc"
tail -c 300 gpurun_out/r02_bench.json
python bench.py --steps 300 --warmup 10 --keyframes-per-step 8 > gpurun_out/r02_bench_c3_g1.json 2> gpurun_out/r02_bench_c3.err; echo "bench c3 rc=$?"
python bench.py --impl reference > gpurun_out/r02_bench_reference.json 2> gpurun_out/r02_bench_reference.err; echo "reference rc=$?"
if [ $rc = 0 ]; then
K='regex:composite|project_|onesweep|adam|loss_|gather_by|emit_|depth_tie|scan_|tile_ranges|order_tiles|grad_gather|expand_kernel'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --launch-skip 400 --launch-count 300 --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_ncu_list.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k "$K" --launch-skip 360 --launch-count 26 -f \
    -o gpurun_out/r02_full python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_ncu_full.log 2>&1; echo "ncu full rc=$?"
fi
