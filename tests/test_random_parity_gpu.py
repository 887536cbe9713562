"""GPU: a bounded run of the randomized parity sweep (scripts/random_parity.py): seeded random
graphs of five families (RMAT permuted / unpermuted, G(n,m), planted cliques, hub clique in a
sparse background) through the C-ABI against the unmodified reference library — truss, nsl and
support bit for bit. The long sweeps of the round are in profiles/r02_random_parity*.log."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))


def test_random_graphs_match_reference(ref):
    r = subprocess.run([sys.executable, os.path.join(ROOT, "scripts", "random_parity.py"), "30", "99"],
                       capture_output=True, text=True, timeout=900, cwd=ROOT)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert "30 graphs, 0 mismatches" in r.stdout
