# compute-sanitizer over the C1-size GPU parity tests: memcheck, racecheck, synccheck.
# Summaries -> gpurun_out/sanitize_<tool>.log (copied to profiles/ by the caller).
SEL='tests/test_gpu_parity.py::test_golden_token_cases tests/test_gpu_parity.py::test_golden_traces_end_to_end
     tests/test_gpu_parity.py::test_row_order_fast_path_and_fallback tests/test_gpu_parity.py::test_streamed_host_names_match_copied_names
     tests/test_gpu_parity.py::test_native_batch_executor_matches_single_trace_calls
     tests/test_gpu_ingest.py::test_adversarial_cases tests/test_op_profile.py::test_device_op_profile_edges
     tests/test_gpu_sa_refine.py::test_full_sa_lcp_vs_reference tests/test_gpu_radix.py::test_sort_pairs_matches_stable_argsort
     tests/test_gpu_batch.py::test_batched_wave_survives_a_failing_trace'
for tool in memcheck racecheck synccheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  [ "$tool" = "racecheck" ] && extra="--racecheck-report hazard"
  timeout 2400 compute-sanitizer --tool $tool $extra --error-exitcode 9 --print-limit 50 \
     python -m pytest $SEL -x -q -p no:cacheprovider -k "not 1000000 and not 3000017 and not 300000 and not 200000" \
     > gpurun_out/sanitize_$tool.log 2>&1
  echo "$tool exit=$?" >> gpurun_out/sanitize_$tool.log
done
