"""Every attention kernel form in the library (RCP_ATTN_VERSION=4: 64-key
blocks; 12: 128-key blocks, 1 CTA; 13 / 14: CTA pairs, alternating blocks /
column-split softmax; 15: v4 with phase-locked tiles; 16: v12 with exp
turn-taking; 17: v12 with the split P arrive) keeps parity
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
    env = dict(os.environ, RCP_ATTN_VERSION=str(version))
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tests", "_variant_check.py")], cwd=ROOT, env=env,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-4000:]
    assert f"version {version}:" in r.stdout
