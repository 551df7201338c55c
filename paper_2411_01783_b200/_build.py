"""Build the in-tree sm_100a extension ``_ringcp_b200.so`` with nvcc.

Run ``python -m paper_2411_01783_b200._build`` (or ``__graft_entry__.build()``).
The library is plain C ABI (include/ringcp_b200.h): no torch types cross it.
"""

from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIB = os.path.join(PKG, "_ringcp_b200.so")
SOURCES = ["capi.cu", "attn_fwd.cu", "attn_fwd_qk8.cu", "decode.cu"]
# The A/B library: the same ABI plus the measured alternative attention forms
# (v12-v17, selected by RCP_ATTN_VERSION).  Not the product:
# loaded only through RCP_LIB_PATH by tests/test_gpu_variants.py and tools/.
LIB_AB = os.path.join(PKG, "_ringcp_b200_ab.so")
SOURCES_AB = SOURCES + ["attn_fwd_n128.cu", "attn_fwd_pair.cu"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.sep not in cand or os.path.exists(cand)):
            return cand
    return "nvcc"


def _start(out: str, sources, extra):
    srcs = [os.path.join(CSRC, s) for s in sources]
    cmd = [nvcc(), *NVCC_FLAGS, *extra, "-I", os.path.join(ROOT, "include"), "-I", CSRC, "-o", out, *srcs]
    return cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)


def build(verbose: bool = False, ab: bool = True) -> str:
    """Build the product library and (``ab``) the A/B library, in parallel."""
    jobs = [("build.log", *_start(LIB, SOURCES, []))]
    if ab:
        jobs.append(("build_ab.log", *_start(LIB_AB, SOURCES_AB, ["-DRCP_AB_FORMS=1"])))
    failed = []
    for log_name, cmd, proc in jobs:
        log = proc.communicate()[0]
        with open(os.path.join(CSRC, log_name), "w") as f:
            f.write(" ".join(cmd) + "\n" + log)
        if verbose:
            print(log)
        if proc.returncode != 0:
            failed.append(f"nvcc failed ({proc.returncode}) for {os.path.basename(cmd[cmd.index('-o') + 1])}:\n"
                          f"{log[-6000:]}")
    if failed:
        raise RuntimeError("\n".join(failed))
    return LIB


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
