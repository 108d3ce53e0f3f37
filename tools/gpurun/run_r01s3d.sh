#!/bin/bash
# Session 3: FlashH2D server after the preload / cache-stream-join fixes.
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_h2d_serve.py tests/test_gpu_pipeline.py -x -q > gpurun_out/s3d_tests.log 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/s3d_smoke.log 2>&1
B="python bench.py --no-cpu-baseline"
timeout 600 $B --hit-trace > gpurun_out/s3d_srv1.json 2> gpurun_out/s3d_srv1.err
timeout 600 $B --h2d-server 0 > gpurun_out/s3d_srv0.json 2> gpurun_out/s3d_srv0.err
timeout 600 $B --slots 262144 > gpurun_out/s3d_slots256k.json 2> gpurun_out/s3d_slots256k.err
timeout 600 $B --groups 4 > gpurun_out/s3d_g4.json 2> gpurun_out/s3d_g4.err
timeout 600 $B --groups 2 > gpurun_out/s3d_g2.json 2> gpurun_out/s3d_g2.err
timeout 600 $B --config C3 > gpurun_out/s3d_c3.json 2> gpurun_out/s3d_c3.err
{ for mu in 4 8 16 32; do echo -n "min_units=$mu "; SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C3; done
  for mu in 8 16; do echo -n "min_units=$mu "; SS_ATTN_MIN_UNITS=$mu python tools/kbench.py attn --cfg C2; done
  for ch in 1024 1824 2048; do echo -n "chunk=$ch "; SS_SEL_CHUNK=$ch python tools/kbench.py select --cfg C3; done
  echo -n "tt1 "; SS_SEL_TT=1 python tools/kbench.py select --cfg C3
} > gpurun_out/s3d_sweeps.txt 2>&1
