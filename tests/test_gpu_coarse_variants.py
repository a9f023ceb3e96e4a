"""The cooperative coarse kernel keeps r and w = A u of a lane group's row pair in shared
memory when every group owns one pair for the whole solve (always on a B200); the global-
memory path it falls back to otherwise must give the same bits.  Each path runs in its own
process (the switch, CHP_C2_NORES, is read once per process)."""

import json
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _hashes(extra_env):
    env = dict(os.environ, **extra_env)
    out = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "coarse_hash.py"), "257"],
                         cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


def test_resident_and_global_cg_vectors_agree_bitwise():
    a = _hashes({})
    b = _hashes({"CHP_C2_NORES": "1"})
    assert a == b
    assert all(v["inc"][0] > 0 for v in a.values())
