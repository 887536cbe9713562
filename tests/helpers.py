"""Shared test helpers: golden fixtures and graph construction (via the oracle's
restatement of the reference test helpers, tests/helpers.hpp:12-43)."""
from __future__ import annotations

import hashlib
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load_fixtures() -> list[dict]:
    with open(os.path.join(GOLDEN, "fixtures.json")) as f:
        return json.load(f)["fixtures"]


def load_configs() -> dict:
    p = os.path.join(GOLDEN, "configs.json")
    if not os.path.exists(p):
        return {}
    with open(p) as f:
        return json.load(f)["configs"]


def build_fixture(oracle, rec):
    """The fixture graph, rebuilt with the oracle's restated generators + canonicalize."""
    rec = rec.get("recipe", rec)
    if rec["kind"] == "er":
        return oracle.er_graph(rec["n"], rec["p"], rec["seed"])
    if rec["kind"] == "rmat":
        return oracle.rmat_graph(rec["scale"], rec["ef"], rec["seed"])
    return oracle.canonicalize(rec["pairs"])


def gpu_graph(csr):
    from paper_1707_02000_b200.trussdec import CsrGraph
    return CsrGraph.from_arrays(csr.offsets, csr.neighbors, csr.labels)
