#!/bin/bash
SS_ATTN_TRACE=1 python tools/kbench.py attn --cfg C3 > gpurun_out/trace_c3.log 2>&1
SS_ATTN_TRACE=1 SS_ATTN_MIN_UNITS=8 python tools/kbench.py attn --cfg C3 >> gpurun_out/trace_c3.log 2>&1
SS_ATTN_TRACE=1 python tools/kbench.py attn --cfg C2 >> gpurun_out/trace_c3.log 2>&1
