#!/bin/bash
# Session 3: FlashH2D server parity + A/B, cache steady state, and the ncu
# evidence pass (reports summarised ON the box, .ncu-rep deleted: gpurun_out <= 64 MiB).
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_h2d_serve.py tests/test_gpu_pipeline.py -x -q > gpurun_out/s3c_tests.log 2>&1
B="python bench.py --no-cpu-baseline"
timeout 600 $B --h2d-server 1 > gpurun_out/s3c_srv1.json 2> gpurun_out/s3c_srv1.err
timeout 600 $B --h2d-server 0 > gpurun_out/s3c_srv0.json 2> gpurun_out/s3c_srv0.err
timeout 600 $B --h2d-server 1 --settle 250 --hit-trace > gpurun_out/s3c_srv1_settle250.json 2> gpurun_out/s3c_srv1_settle250.err
timeout 600 $B --h2d-server 1 --settle 250 --slots 262144 > gpurun_out/s3c_srv1_slots256k.json 2> gpurun_out/s3c_srv1_slots256k.err
timeout 600 $B --h2d-server 1 --groups 4 > gpurun_out/s3c_srv1_g4.json 2> gpurun_out/s3c_srv1_g4.err
timeout 600 $B --h2d-server 1 --config C3 > gpurun_out/s3c_srv1_c3.json 2> gpurun_out/s3c_srv1_c3.err
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
# --settle 10 --warmup 3: 13 eager steps x 576 launches (3 groups x 32 layers x 6) precede the timed step
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 7488 -c 576 --csv \
   --log-file gpurun_out/s3c_launches.csv $B --h2d-server 0 --steps 1 --warmup 3 --settle 10 --no-gather-alone > gpurun_out/s3c_ncu_list.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k "$KR" -s 7488 -c 6 \
   -o /tmp/s3c_step $B --h2d-server 0 --steps 1 --warmup 3 --settle 10 --no-gather-alone > gpurun_out/s3c_ncu_full.log 2>&1
python tools/ncu_summary.py /tmp/s3c_step.ncu-rep > gpurun_out/s3c_ncu_step_summary.txt 2>&1
ncu -i /tmp/s3c_step.ncu-rep --page raw --csv > gpurun_out/s3c_ncu_step_raw.csv 2>/dev/null
for cfg in C2 C3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 3 -c 1 \
     -o /tmp/s3c_attn_$cfg python tools/kbench.py attn --cfg $cfg --iters 2 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select -s 3 -c 1 \
     -o /tmp/s3c_sel_$cfg python tools/kbench.py select --cfg $cfg --iters 2 > /dev/null 2>&1
  for k in attn sel; do
    python tools/ncu_summary.py /tmp/s3c_${k}_$cfg.ncu-rep > gpurun_out/s3c_ncu_${k}_$cfg.txt 2>&1
    ncu -i /tmp/s3c_${k}_$cfg.ncu-rep --page source --csv --print-source sass > /tmp/src_${k}_$cfg.csv 2>/dev/null
    python tools/ncu_source_hot.py /tmp/src_${k}_$cfg.csv 40 > gpurun_out/s3c_hot_${k}_$cfg.txt 2>&1
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum \
   --clock-control none -k regex:flash_h2d -s 2 -c 3 --csv --log-file gpurun_out/s3c_gather_pcie.csv \
   python tools/kbench.py gather --iters 2 > gpurun_out/s3c_gather_pcie.log 2>&1
du -sh gpurun_out
