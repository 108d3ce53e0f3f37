#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck, initcheck) over the C1-sized
# parity suites of every kernel family: select (atomic-ticket merge), cache
# (grid-wide last-CTA plans), gather, attention (stream-K tickets, TMA/mbarrier),
# the FlashH2D server + flag protocol (spin-waits), meta update, and one
# request-group pipeline step sequence (server + graph).
mkdir -p gpurun_out/sanitize
SEL='test_select_c1_shape or test_select_gqa_ragged_multichunk or test_select_ties_and_k_edges or test_cache_multistep_bit_exact or test_cache_hand_traced_fixture or test_cache_invalid_key or test_flash_h2d_gather_byte_exact or test_attention_tolerance or test_attention_empty_and_tail_only or test_attention_many_pairs_stream_k or test_attention_skipped_on_error_status or test_block_meta_update_bit_exact or test_attention_split_hits_misses_merge'
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ "$tool" = "memcheck" ] && extra="--leak-check no"
  timeout 1500 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
      python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "$SEL" \
      > gpurun_out/sanitize/${tool}_parity.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitize/${tool}_parity.log
  timeout 900 compute-sanitizer --tool $tool $extra --target-processes all --print-limit 50 \
      python -m pytest -q -x -p no:cacheprovider tests/test_gpu_h2d_serve.py -k "byte_exact or reused or stats" \
      > gpurun_out/sanitize/${tool}_h2d_serve.log 2>&1
  echo "exit=$?" >> gpurun_out/sanitize/${tool}_h2d_serve.log
done
timeout 1500 compute-sanitizer --tool memcheck --leak-check no --target-processes all --print-limit 50 \
    python -m pytest -q -x -p no:cacheprovider "tests/test_gpu_pipeline.py::test_request_groups_pipeline_two_streams[4-True-3-False-True]" \
    > gpurun_out/sanitize/memcheck_pipeline_groups.log 2>&1
echo "exit=$?" >> gpurun_out/sanitize/memcheck_pipeline_groups.log
