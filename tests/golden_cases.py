"""Loader for the committed golden fixtures (tests/golden/, made by make_golden.py
from the reference itself)."""
from __future__ import annotations

import json
import os
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
GOLDEN = os.path.join(HERE, "golden")

PREC_NAMES = ("fp64", "fp32", "fp16")


def load_configs() -> dict:
    with open(os.path.join(GOLDEN, "golden.json")) as f:
        return json.load(f)["configs"]


@dataclass
class Case:
    meta: dict
    x: list
    rel: list
    cell: list
    items: np.ndarray
    start: np.ndarray
    cell_of: np.ndarray
    tables: dict = field(default_factory=dict)

    @property
    def name(self):
        return self.meta["name"]

    @property
    def dim(self):
        return self.meta["dim"]

    @property
    def n(self):
        return self.meta["n"]

    def table(self, backend: str, prec: str):
        return self.tables[f"{backend}_{prec}"]


_cases = None


def load_cases() -> list:
    global _cases
    if _cases is None:
        with open(os.path.join(GOLDEN, "small_cases.json")) as f:
            index = json.load(f)
        z = np.load(os.path.join(GOLDEN, "small_cases.npz"))
        out = []
        for m in index:
            k, d = m["key"], m["dim"]
            c = Case(m, [z[f"{k}_x{a}"] for a in range(d)], [z[f"{k}_rel{a}"] for a in range(d)],
                     [z[f"{k}_cell{a}"] for a in range(d)], z[f"{k}_items"], z[f"{k}_start"],
                     z[f"{k}_cellof"])
            for be in ("rcll", "cll", "all"):
                for p in PREC_NAMES:
                    c.tables[f"{be}_{p}"] = (z[f"{k}_{be}_{p}_off"], z[f"{k}_{be}_{p}_items"])
            out.append(c)
        _cases = out
    return _cases
