#!/bin/bash
# Round-2 evidence for profiles/: the bench line, ncu launch list, one ncu --set full capture
# of a mapping step (each only after the plain command exited 0), then the C5 stress run.
set -u
python bench.py --steps 300 --warmup 10 > gpurun_out/r02_bench.json 2> gpurun_out/r02_bench.err; echo "bench rc=$?"
tail -c 400 gpurun_out/r02_bench.json
K='regex:composite|project_|onesweep|adam|loss_|gather_by|emit_|depth_tie|scan_|tile_ranges|order_tiles|grad_gather|expand_kernel'
ncu --metrics gpu__time_duration.sum --clock-control none -k "$K" --launch-skip 400 --launch-count 300 --csv \
    --log-file gpurun_out/r02_launches.csv python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_ncu_list.log 2>&1; echo "ncu list rc=$?"
ncu --set full --clock-control none --import-source on -k "$K" --launch-skip 360 --launch-count 26 -f \
    -o gpurun_out/r02_full python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02_ncu_full.log 2>&1; echo "ncu full rc=$?"
bash tools/stream_runs.sh 2>&1 | grep c5
