#!/bin/sh
# Build the RCP_TRACE variant of the library used by tools/trace_attn.py.
# Usage: tools/build_trace.sh [output-name] [extra nvcc flags...]
out=${1:-_ringcp_b200_trace.so}
[ $# -gt 0 ] && shift
cd "$(dirname "$0")/../paper_2411_01783_b200/csrc" && nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -DRCP_TRACE=1 -DRCP_TRACE_BUILD -DRCP_AB_FORMS=1 "$@" -I../../include -I. -o ../$out capi.cu attn_fwd.cu attn_fwd_n128.cu attn_fwd_pair.cu decode.cu
