"""GPU: the checked build (-DTDG_CHECKS=1: device-side bounds / invariant checks that trap on
violation, tdg_common.cuh TDG_CHECK) over every golden fixture, the hand-built step states,
the edge-list parser and BASELINE configs 1 and 3, each compared with the reference goldens.
compute-sanitizer is closed on the GPU pool, so this is the memory-safety run."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
CHECKED = os.path.join(ROOT, "paper_1707_02000_b200", "lib_variants", "checked", "libtdg.so")


def _run(args, timeout):
    assert os.path.exists(CHECKED), "checked build missing (__graft_entry__.build() makes it)"
    env = dict(os.environ, TDG_SO=CHECKED)
    return subprocess.run([sys.executable] + args, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)


def test_checked_build_fixtures_steps_parser_c1():
    r = _run([os.path.join(ROOT, "scripts", "sanitize.py")], 900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert "0 mismatches" in r.stdout


def test_checked_build_config3():
    r = _run([os.path.join(ROOT, "scripts", "run_one.py"), "3", "1"], 900)
    assert r.returncode == 0, (r.stdout + r.stderr)[-3000:]
    assert "parity=ok" in r.stdout and "checked" in r.stdout
