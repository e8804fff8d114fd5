# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over small
# batches of every kernel: every K1 engine (lane v7 incl. its retry pass and
# in-kernel exact fallback, octet v8 incl. its fallback, step-program lane
# v6, warp v3), the host pipeline with K5 pack16, step programs, float64 mode, event
# logs, CSR batches, K2-K4.  Logs -> gpurun_out/sanitize_<tool>.log
mkdir -p gpurun_out
SEL="golden_burst or golden_multidev or edge_cases or lane_fallback or lane_retry_pass or many_priority_classes or ragged_offsets or generator_bit_identical or reduce_stats or select_grants_batch_golden or bad_device or octet_kernel or host_pipeline_cases or program_batches"
DROP="readme or mixed or 4799"
for tool in ${TOOLS:-memcheck synccheck racecheck initcheck}; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout ${SAN_TIMEOUT:-900} compute-sanitizer --tool $tool $extra --print-limit 100 --error-exitcode 99 \
      python -m pytest tests/test_gpu_parity.py tests/test_gpu_dropin.py -q -x -p no:cacheprovider \
      -k "($SEL) or (test_report_matches_reference and ($DROP))" \
      > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool rc=$?"
  grep -E "ERROR SUMMARY|passed|failed" gpurun_out/sanitize_$tool.log | tail -3
done
