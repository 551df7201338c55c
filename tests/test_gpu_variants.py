"""Every attention kernel form of the A/B library (_ringcp_b200_ab.so, built
next to the product library by build(); the product library has only v4):
RCP_ATTN_VERSION=4: 64-key blocks; 12: 128-key blocks, 1 CTA; 13 / 14: CTA pairs, alternating blocks /
column-split softmax; 15: v4 with phase-locked tiles; 16: v12 with exp
turn-taking; 17: v12 with the split P arrive.  Each keeps parity
with the fp32 reference: each runs in a fresh process (the library reads the
selector once) on eight random segmented / GQA / merge cases
(tests/_variant_check.py)."""

import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("version", [4, 12, 13, 14, 15, 16, 17])
def test_variant_parity(version):
    lib = os.path.join(ROOT, "paper_2411_01783_b200", "_ringcp_b200_ab.so")
    assert os.path.exists(lib), "A/B library not built (paper_2411_01783_b200._build.build(ab=True))"
    env = dict(os.environ, RCP_ATTN_VERSION=str(version), RCP_LIB_PATH=lib)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_variant_check.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert f"version {version}:" in r.stdout
