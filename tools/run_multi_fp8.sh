# FP8 (e4m3) KV decode on 2 / 4 GPUs: eager-vs-graph agreement over NCCL and the cfg5 graphed step.
cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NG=$(nvidia-smi -L | wc -l)
GD_KV=e4m3 GD_TABLE=1 GD_GROUPED=1 timeout 600 $TR --nproc-per-node $NG --master-port 29511 tools/decode_graph_check.py > gpurun_out/m_dgc_fp8.log 2>&1; grep "world" gpurun_out/m_dgc_fp8.log; tail -2 gpurun_out/m_dgc_fp8.log
for dt in bf16 e4m3; do
timeout 600 $TR --nproc-per-node $NG --master-port 2952$NG tools/bench_configs.py decode --graph --context 1048576 --batch 1 4 32 --steps 20 --warmup 3 --kv-dtype $dt > gpurun_out/m_cfg5_cp${NG}_$dt.jsonl 2> gpurun_out/m_cfg5_$dt.err; cat gpurun_out/m_cfg5_cp${NG}_$dt.jsonl; tail -2 gpurun_out/m_cfg5_$dt.err
done
