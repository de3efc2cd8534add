"""Seeded synthetic knowledge graphs shaped like the paper's datasets (input generation only).

Shapes follow PAPER.md Table 3 (L629-640) as restated in BASELINE.json configs; the degree / relation-frequency
law (Zipf with alpha_e=0.8, alpha_r=1.0) is a proposal (the paper gives no such statistics -- "parity unpinned"
for workload realism). This module holds none of the method's arithmetic.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

from .build import LIB
from .build import build as build_lib

GRAPH_SEED = 0x20040853


class _Graph(ctypes.Structure):
    _fields_ = [("n_entities", ctypes.c_int64), ("n_relations", ctypes.c_int64), ("n_triples", ctypes.c_int64),
                ("alpha_e", ctypes.c_double), ("alpha_r", ctypes.c_double), ("graph_seed", ctypes.c_uint64)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            build_lib()
        _lib = ctypes.CDLL(LIB)
        P = ctypes.POINTER
        _lib.synth_triple.argtypes = [P(_Graph), ctypes.c_int64, P(ctypes.c_int64), P(ctypes.c_int64), P(ctypes.c_int64)]
        _lib.synth_triples.argtypes = [P(_Graph), ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p, ctypes.c_void_p,
                                       ctypes.c_void_p]
        _lib.synth_triples_i32.argtypes = _lib.synth_triples.argtypes
    return _lib


@dataclass
class Graph:
    name: str
    n_entities: int
    n_relations: int
    n_triples: int
    alpha_e: float = 0.8
    alpha_r: float = 1.0
    graph_seed: int = GRAPH_SEED

    def _c(self) -> _Graph:
        return _Graph(self.n_entities, self.n_relations, self.n_triples, self.alpha_e, self.alpha_r, self.graph_seed)

    def triples(self, begin: int = 0, n: int | None = None, dtype=np.int64):
        """(h, r, t) arrays for triples [begin, begin+n)."""
        n = self.n_triples - begin if n is None else n
        h = np.empty(n, dtype=dtype)
        r = np.empty(n, dtype=dtype)
        t = np.empty(n, dtype=dtype)
        fn = lib().synth_triples if dtype == np.int64 else lib().synth_triples_i32
        g = self._c()
        fn(ctypes.byref(g), begin, n, h.ctypes.data, r.ctypes.data, t.ctypes.data)
        return h, r, t

    def triple(self, i: int):
        g = self._c()
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        lib().synth_triple(ctypes.byref(g), i, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
        return a.value, b.value, c.value


# BASELINE.json configs[0..4]
GRAPHS = {
    "tiny": Graph("tiny", 1_000, 20, 10_000),
    "fb15k": Graph("fb15k", 14_951, 1_345, 483_142),
    "wn18": Graph("wn18", 40_943, 18, 141_442),
    "freebase": Graph("freebase", 86_054_151, 14_824, 338_586_276),
}


def graph(name: str, **overrides) -> Graph:
    g = GRAPHS[name]
    if overrides:
        d = dict(g.__dict__)
        d.update(overrides)
        return Graph(**d)
    return g
