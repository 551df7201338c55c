# Bound-finding builds of the library (not the product): S over half the K-dim,
# no exponentials.  Loaded with RCP_LIB_PATH=tools/_dbg/<name>.so.
set -e
cd "$(dirname "$0")/.."
P=paper_2411_01783_b200/csrc
SRC="$P/capi.cu $P/attn_fwd.cu $P/attn_fwd_n128.cu $P/attn_fwd_pair.cu $P/decode.cu"
F="-gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -Xcompiler -fPIC -shared -I include -I $P -DRCP_AB_FORMS=1"
nvcc $F -DRCP_DBG_S_STEPS=4 -o tools/_dbg/half_s.so $SRC
nvcc $F -DRCP_DBG_NO_EXP=1 -o tools/_dbg/no_exp.so $SRC
nvcc $F -DRCP_DBG_S_STEPS=4 -DRCP_DBG_NO_EXP=1 -o tools/_dbg/half_s_no_exp.so $SRC
# exp2 split of the 128-key forms (v12 / v16): pairs of every 8 on the FMA-pipe polynomial
nvcc $F -DRCP_POLY_PAIRS_N=3 -o tools/_dbg/poly3.so $SRC
nvcc $F -DRCP_POLY_PAIRS_N=4 -o tools/_dbg/poly4.so $SRC
