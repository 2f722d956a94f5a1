#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the C1-size
# GPU parity tests, our kernels only (the sm:: namespace).  Logs -> gpurun_out/.
#   bash tools/sanitize.sh
set -u
CS=/usr/local/cuda/bin/compute-sanitizer
TESTS="tests/test_render_gpu.py::test_forward_matches_reference_golden tests/test_render_gpu.py::test_known_answers tests/test_render_gpu.py::test_backward_matches_oracle tests/test_render_gpu.py::test_edge_cases_match_oracle tests/test_render_gpu.py::test_loss_gradient_matches_oracle tests/test_binning_gpu.py::test_binning_edge_cases_bit_exact tests/test_mapping_gpu.py::test_graph_replay_equals_eager tests/test_mapping_gpu.py::test_adam_kernel_matches_oracle tests/test_store_gpu.py::test_evict_reload_bit_exact_with_adam_state tests/test_sample_gpu.py::test_lift_matches_reference tests/test_loopclose_gpu.py::test_reference_properties"
mkdir -p gpurun_out
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = racecheck ] && extra="--racecheck-report all"
  timeout 1500 $CS --tool $tool $extra --kernel-name regex:sm:: --print-limit 50 --error-exitcode 9 \
    python -m pytest -q -p no:cacheprovider $TESTS > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY|passed|failed' gpurun_out/sanitize_$tool.log | tail -3 | tr '\n' ' ')"
done
