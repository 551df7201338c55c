cd $GRAFT_REPO_ROOT
TR="python -m torch.distributed.run --nnodes=1 --master-addr 127.0.0.1"
timeout 600 python -m pytest tests/test_gpu_multi_fused_a2a.py -q 2>&1 | tail -2
timeout 600 $TR --nproc-per-node 2 --master-port 29501 bench.py --gpus 2 --steps 10 --warmup 3 --check > gpurun_out/m_bench_cp2.jsonl 2> gpurun_out/m_bench_cp2.err; tail -c 1500 gpurun_out/m_bench_cp2.jsonl; tail -3 gpurun_out/m_bench_cp2.err
timeout 600 $TR --nproc-per-node 4 --master-port 29502 bench.py --gpus 4 --steps 10 --warmup 3 --check > gpurun_out/m_bench_cp4.jsonl 2> gpurun_out/m_bench_cp4.err; tail -c 1500 gpurun_out/m_bench_cp4.jsonl; tail -3 gpurun_out/m_bench_cp4.err
timeout 900 $TR --nproc-per-node 4 --master-port 29503 bench.py --gpus 4 --config 405b --steps 5 --warmup 3 --check --no-e2e > gpurun_out/m_bench_cp4_405b.jsonl 2> gpurun_out/m_bench_cp4_405b.err; tail -c 1200 gpurun_out/m_bench_cp4_405b.jsonl
timeout 600 $TR --nproc-per-node 4 --master-port 29504 tools/bench_configs.py decode --graph --context 1048576 --batch 1 4 32 --steps 20 --warmup 3 > gpurun_out/m_cfg5_cp4_table.jsonl 2> gpurun_out/m_cfg5.err; cat gpurun_out/m_cfg5_cp4_table.jsonl; tail -3 gpurun_out/m_cfg5.err
timeout 600 $TR --nproc-per-node 4 --master-port 29505 tools/bench_configs.py decode --graph --no-table --context 1048576 --batch 1 --steps 20 --warmup 3 > gpurun_out/m_cfg5_cp4_upload.jsonl 2>&1; tail -2 gpurun_out/m_cfg5_cp4_upload.jsonl
timeout 900 $TR --nproc-per-node 4 --master-port 29506 tools/bench_configs.py partial --calibrate --steps 5 --warmup 2 > gpurun_out/m_cfg4_cp4_calibrated.jsonl 2> gpurun_out/m_cfg4.err; cat gpurun_out/m_cfg4_cp4_calibrated.jsonl; tail -3 gpurun_out/m_cfg4.err
timeout 600 $TR --nproc-per-node 4 --master-port 29507 tools/ring_nccl_check.py > gpurun_out/m_ring_nccl_check4.log 2>&1; tail -5 gpurun_out/m_ring_nccl_check4.log
