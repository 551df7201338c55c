"""CPU: the bench's contract pieces that do not need a GPU — both arms share
one config object, the ragged fused-batch split, the reference-arm sample
bookkeeping, and the command-line flags the driver and DESIGN.md use."""

import json
import subprocess
import sys

import pytest

import bench


@pytest.mark.parametrize("K", [1, 3, 7])
def test_ragged_seq_lens_cover_T(K):
    T = bench.CONFIGS["8b"]["T"]
    lens = bench.ragged_seq_lens(T, K)
    assert len(lens) == K and sum(lens) == T and all(x > 0 for x in lens)
    assert lens == sorted(lens)  # 1 : 2 : ... : K


def test_workload_config_is_shared_and_labelled():
    for name, cfg in bench.CONFIGS.items():
        for world in (1, 2, 4, 8):
            c = bench.workload_config(cfg, world, 1)
            assert c["workload"] == cfg["workload"] and c["seq_len"] == cfg["T"]
            assert c["cp"] == world and c["parallelism"] == f"cp{world}" and c["protocol"] == "pass_kv"
            assert "inputs larger than L2" in c["l2"]
            json.dumps(c)
    assert "seq_lens" in bench.workload_config(bench.CONFIGS["8b"], 1, 3)


def test_cfg1_inputs_are_bf16_exact():
    import numpy as np

    q, k, v = bench._cfg1_inputs()
    assert q.shape == (4096, 8, 128) and k.shape == (4096, 1, 128) and v.shape == (4096, 1, 128)
    for x in (q, k, v):
        assert np.all((x.view(np.uint32) & 0xFFFF) == 0)  # bf16-representable


def test_cli_flags_parse():
    out = subprocess.run([sys.executable, "bench.py", "--help"], capture_output=True, text=True, timeout=120)
    assert out.returncode == 0
    for flag in ("--gpus", "--steps", "--warmup", "--impl", "--config", "--seq-len", "--seqs", "--no-e2e",
                 "--check", "--e2e-ranges", "--fp8-qk", "--no-cfg1", "--no-cpu-baseline"):
        assert flag in out.stdout, flag
