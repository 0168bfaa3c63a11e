# compute-sanitizer passes over the small GPU parity cases (run through gpurun
# from the repo root): memcheck (out-of-bounds / misaligned global, shared and
# TMA accesses), synccheck (barrier misuse), racecheck (shared-memory hazards)
# and initcheck (reads of device memory nobody wrote).  The tests still compare
# with the oracle, so a pass is "parity green and no sanitizer error".
S="compute-sanitizer --error-exitcode 86 --print-limit 20"
# ragged / degenerate shapes, every BC, the three correction forms, several
# flips per layer, LAZY, offline + partial re-execution, slab groups (fused halo)
K1="cfg1_online or ragged or fig2 or tile_and_chunk or bc_hotspot or multi_flip or recompute_layer_ragged or partial_reexecution or lazy_many or slab_group_equals_oracle or last_window_shorter or generic_stencil"
K2="cfg1_online or hotspot_ragged or multi_flip or lazy_many or last_window_shorter or (partial_reexecution and 3) or (slab_group_equals_oracle and 2-False)"
run() {  # name, tool options, pytest -k expression, files
  local name=$1 opts=$2 k=$3; shift 3
  timeout 1200 $S $opts python -m pytest "$@" -m gpu -q -x -k "$k" > gpurun_out/sanitize_$name.log 2>&1
  echo "${name}_rc=$?"
  grep -E "ERROR SUMMARY|passed|failed|RACECHECK SUMMARY" gpurun_out/sanitize_$name.log | tail -4
}
run memcheck "--tool memcheck" "$K1" tests/test_gpu_parity.py
run memcheck_pipeline "--tool memcheck" "graph_replays or layer_recompute or many_rewrites or plan_then or consecutive_flips" tests/test_gpu_pipeline.py
run synccheck "--tool synccheck" "$K2" tests/test_gpu_parity.py
run racecheck "--tool racecheck --racecheck-report analysis" "$K2" tests/test_gpu_parity.py
run initcheck "--tool initcheck" "$K2" tests/test_gpu_parity.py
