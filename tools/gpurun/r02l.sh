#!/bin/bash
# Round 2: attention with deferred merges (after the warp's own range) and a
# wider merge load batch -- parity, kernels alone (group shape, full C2, C3),
# per-warp timelines, the C2 step.
mkdir -p gpurun_out/r02l
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_pipeline.py -q -k "attention or fullsize or c1_pipeline or request_groups" > gpurun_out/r02l/tests.log 2>&1
echo "rc=$?" >> gpurun_out/r02l/tests.log
{
for a in "--cfg C2 --batch 3" "--cfg C2 --batch 4" "--cfg C2" "--cfg C3"; do
  echo "$a $(python tools/kbench.py attn $a)"
done
for ns in 3 4; do for mu in 8 16 32; do
  echo "stages=$ns min_units=$mu batch3 $(SS_LIB_VARIANT=debug SS_ATTN_STAGES=$ns SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C2 --batch 3)"
  echo "stages=$ns min_units=$mu C3 $(SS_LIB_VARIANT=debug SS_ATTN_STAGES=$ns SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C3)"
done; done
SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 python tools/kbench.py attn --cfg C2 --batch 3
SS_LIB_VARIANT=debug SS_ATTN_TRACE=1 python tools/kbench.py attn --cfg C3
} > gpurun_out/r02l/kbench_attn.txt 2>&1
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r02l/bench_c2.json 2> gpurun_out/r02l/bench_c2.err
# initcheck attribution: kernel-side reads vs host copies of partly written buffers
SEL='test_select_c1_shape or test_select_gqa_ragged_multichunk or test_cache_multistep_bit_exact or test_flash_h2d_gather_byte_exact or test_attention_tolerance or test_block_meta_update_bit_exact'
timeout 1200 compute-sanitizer --tool initcheck --target-processes all --print-limit 100000 \
    python -m pytest -q -x -p no:cacheprovider tests/test_gpu_parity.py -k "$SEL" > gpurun_out/r02l/initcheck_full.log 2>&1
grep -c "on access by cudaMemcpy" gpurun_out/r02l/initcheck_full.log > gpurun_out/r02l/initcheck_counts.txt
grep -c "by thread" gpurun_out/r02l/initcheck_full.log >> gpurun_out/r02l/initcheck_counts.txt
grep -A3 "by thread" gpurun_out/r02l/initcheck_full.log | grep -E "at .* in " | sed -E 's/.* in ([^ ]*).*/\1/' | sort | uniq -c >> gpurun_out/r02l/initcheck_counts.txt
gzip -9 gpurun_out/r02l/initcheck_full.log
