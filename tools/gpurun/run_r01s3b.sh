#!/bin/bash
# Session 3: cache steady state (settle length, cache size) and the ncu evidence
# pass of the current kernels (launch list of one graph-replayed step + full
# captures of its first 6 hot-path launches + select/attention alone).
mkdir -p gpurun_out
B="python bench.py --no-cpu-baseline"
timeout 600 $B --settle 250 --hit-trace > gpurun_out/s3b_settle250.json 2> gpurun_out/s3b_settle250.err
timeout 600 $B --settle 250 --slots 262144 --hit-trace > gpurun_out/s3b_slots256k.json 2> gpurun_out/s3b_slots256k.err
timeout 600 $B --settle 250 --slots 196608 > gpurun_out/s3b_slots192k.json 2> gpurun_out/s3b_slots192k.err
KR='regex:block_select|cache_|flash_h2d|sparse_attn'
# --settle 10 --warmup 3: 13 eager steps x 576 launches (3 groups x 32 layers x 6) precede the timed step
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k "$KR" -s 7488 -c 576 --csv \
   --log-file gpurun_out/s3b_launches.csv $B --steps 1 --warmup 3 --settle 10 --no-gather-alone > gpurun_out/s3b_ncu_list.log 2>&1
timeout 1800 ncu --set full --clock-control none --import-source on -k "$KR" -s 7488 -c 6 \
   -o gpurun_out/s3b_step $B --steps 1 --warmup 3 --settle 10 --no-gather-alone > gpurun_out/s3b_ncu_full.log 2>&1
for cfg in C2 C3; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:sparse_attn -s 3 -c 1 \
     -o gpurun_out/s3b_attn_$cfg python tools/kbench.py attn --cfg $cfg --iters 2 > /dev/null 2>&1
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:block_select -s 3 -c 1 \
     -o gpurun_out/s3b_sel_$cfg python tools/kbench.py select --cfg $cfg --iters 2 > /dev/null 2>&1
done
timeout 600 ncu --set full --clock-control none -k regex:flash_h2d -s 2 -c 1 \
   -o gpurun_out/s3b_gather python tools/kbench.py gather --iters 2 > /dev/null 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum,pcie__read_bytes.sum,pcie__write_bytes.sum,dram__bytes_read.sum,dram__bytes_write.sum,syslts__d_sectors_fill_sysmem.sum \
   --clock-control none -k regex:flash_h2d -s 2 -c 3 --csv --log-file gpurun_out/s3b_gather_pcie.csv \
   python tools/kbench.py gather --iters 2 > /dev/null 2>&1
