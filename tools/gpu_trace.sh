#!/bin/bash
mkdir -p gpurun_out
export SD_ATTN_TRACE=1
( python tools/trace_umma.py 4096 128 5; python tools/trace_umma.py 8192 128 5; python tools/trace_umma.py 4608 26 5;
  python tools/trace_umma.py 4608 102 0 230; python tools/trace_umma.py 32768 128 5 ) > gpurun_out/trace.log 2>&1
