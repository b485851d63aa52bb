"""Loader for the committed golden fixtures (see tests/golden/make_golden.py)."""

from __future__ import annotations

import json
from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def manifest():
    return json.loads((GOLDEN / "manifest.json").read_text())


@lru_cache(maxsize=None)
def fused():
    return dict(np.load(GOLDEN / "fused_golden.npz"))


@lru_cache(maxsize=None)
def solvers():
    return dict(np.load(GOLDEN / "solver_golden.npz"))


def csr_arrays(store, key):
    shape = store[f"{key}/shape"]
    return int(shape[0]), int(shape[1]), store[f"{key}/rowptr"], store[f"{key}/cols"], store[f"{key}/vals"]


def solver_case(name):
    for case in manifest()["solver_cases"]:
        if case["name"] == name:
            return case
    raise KeyError(name)


def solver_case_names():
    return [c["name"] for c in manifest()["solver_cases"]]


@lru_cache(maxsize=None)
def classical():
    return dict(np.load(GOLDEN / "classical_golden.npz"))


def classical_case(name):
    for case in manifest()["classical_cases"]:
        if case["name"] == name:
            return case
    raise KeyError(name)


def classical_case_names():
    return [c["name"] for c in manifest()["classical_cases"]]
