# The round-2 multi-GPU evidence run on all GPUs of the box (2 or 4): CP bench
# with the parity check, 405B shape, cfg5 decode (p2p and NCCL transports,
# bf16 and e4m3 KV), cfg4 with the calibrated heuristic, NCCL ring check.
cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
NG=$(nvidia-smi -L | wc -l)
timeout 600 python -m pytest tests/test_gpu_multi_fused_a2a.py tests/test_gpu_multi_p2p_decode.py -q 2>&1 | tail -2
timeout 600 $TR --nproc-per-node 2 --master-port 29501 bench.py --gpus 2 --steps 10 --warmup 3 --check --no-cfg1 > gpurun_out/m_bench_cp2.jsonl 2> gpurun_out/m_bench_cp2.err; tail -c 600 gpurun_out/m_bench_cp2.jsonl; tail -3 gpurun_out/m_bench_cp2.err
if [ "$NG" -ge 4 ]; then
timeout 600 $TR --nproc-per-node 4 --master-port 29502 bench.py --gpus 4 --steps 10 --warmup 3 --check --no-cfg1 > gpurun_out/m_bench_cp4.jsonl 2> gpurun_out/m_bench_cp4.err; tail -c 600 gpurun_out/m_bench_cp4.jsonl; tail -3 gpurun_out/m_bench_cp4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29503 bench.py --gpus 4 --config 405b --steps 5 --warmup 3 --check --no-e2e --no-cfg1 > gpurun_out/m_bench_cp4_405b.jsonl 2> gpurun_out/m_bench_cp4_405b.err; tail -c 600 gpurun_out/m_bench_cp4_405b.jsonl
fi
for KV in bf16 e4m3; do for T in p2p nccl; do
timeout 300 $TR --nproc-per-node $NG --master-port 2957$NG tools/bench_configs.py decode --graph --context 1048576 --batch 1 4 32 --steps 20 --warmup 3 --kv-dtype $KV --transport $T > gpurun_out/m_cfg5_${T}_$KV.jsonl 2> gpurun_out/m_cfg5_${T}_$KV.err; cat gpurun_out/m_cfg5_${T}_$KV.jsonl
done; done
timeout 900 $TR --nproc-per-node $NG --master-port 29506 tools/bench_configs.py partial --calibrate --steps 5 --warmup 2 > gpurun_out/m_cfg4_calibrated.jsonl 2> gpurun_out/m_cfg4.err; cat gpurun_out/m_cfg4_calibrated.jsonl; tail -3 gpurun_out/m_cfg4.err
timeout 600 $TR --nproc-per-node $NG --master-port 29507 tools/ring_nccl_check.py > gpurun_out/m_ring_nccl_check.log 2>&1; tail -5 gpurun_out/m_ring_nccl_check.log
