"""Randomised parity sweep (tools/fuzz_parity.py): random batch sizes, node counts, run modes and
group plans, start modes, force models, spreads and iteration caps -- device vs the CPU oracle,
same exception or agreement within the north-star bars."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("seed", [3, 101])
def test_fuzz_parity(seed):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "fuzz_parity.py"), "60", str(seed)],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert r.stdout.strip().splitlines()[-1].endswith(" 0 mismatches"), r.stdout[-4000:]
