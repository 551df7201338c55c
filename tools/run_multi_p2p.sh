# Decode step transport A/B on all GPUs of the box: NCCL collectives vs kernel
# stores into CUDA-IPC peer buffers (GraphedDecode(transport="p2p")).
cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NG=$(nvidia-smi -L | wc -l)
for T in p2p nccl; do
GD_TRANSPORT=$T GD_TABLE=1 GD_GROUPED=1 timeout 300 $TR --nproc-per-node $NG --master-port 2956$NG tools/decode_graph_check.py > gpurun_out/m_dgc_$T.log 2>&1; grep "world" gpurun_out/m_dgc_$T.log; grep -i "error\|Traceback" gpurun_out/m_dgc_$T.log | head -3
done
for KV in bf16 e4m3; do for T in p2p nccl; do
timeout 300 $TR --nproc-per-node $NG --master-port 2957$NG tools/bench_configs.py decode --graph --context 1048576 --batch 1 4 32 --steps 20 --warmup 3 --kv-dtype $KV --transport $T > gpurun_out/m_cfg5_${T}_$KV.jsonl 2> gpurun_out/m_cfg5_${T}_$KV.err; cat gpurun_out/m_cfg5_${T}_$KV.jsonl; grep -i "error\|Traceback" gpurun_out/m_cfg5_${T}_$KV.err | head -3
done; done
