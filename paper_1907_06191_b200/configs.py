"""Seeded synthetic workloads c1..c5 (BASELINE.json "configs").

Input recipes only (no method arithmetic).  Grid units: h = 1 pixel, D = 1;
the physical mapping is h = 0.125 um, D = 450 um^2/s, so one
time unit is h^2/D = 34.72 us.
"""
from __future__ import annotations

from dataclasses import dataclass
from functools import lru_cache

import numpy as np

from . import substrate as S


@dataclass(frozen=True)
class Config:
    name: str
    n: int                 # grid n x n
    degree: int
    dt: float
    nsteps: int
    n_sources: int
    describe: str


CONFIGS = {
    "c1": Config("c1", 32, 1, 1 / 32, 200, 1, "32x32, one centred disk r=8 px, 1 source (4,16), P1"),
    "c2": Config("c2", 256, 1, 1 / 32, 512, 1024, "256x256 free, 1024 lattice sources, P1 (closed form)"),
    "c3": Config("c3", 512, 1, 1 / 32, 256, 4096, "512x512 Gamma f=0.60 seed 3, 4096 sources seed 4, P1"),
    "c4": Config("c4", 2048, 1, 1 / 32, 32, 65536, "2048x2048 Gamma f=0.60 seed 5, 65536 sources seed 6, P1"),
    "c5": Config("c5", 1024, 2, 1 / 128, 100000, 64, "1024x1024 Gamma f=0.60 seed 7, 64 sources seed 8, P2"),
}

SUBSTRATE_SEED = {"c3": 3, "c4": 5, "c5": 7}
SOURCE_SEED = {"c3": 4, "c4": 6, "c5": 8}


@lru_cache(maxsize=8)
def mask(name: str) -> np.ndarray:
    c = CONFIGS[name]
    if name == "c1":
        m = S.disk_substrate(32, 16.0, 16.0, 8.0)
    elif name == "c2":
        m = np.zeros((256, 256), np.uint8)
    else:
        m = S.gen_substrate(c.n, c.n, 0.60, SUBSTRATE_SEED[name]).mask
    m.setflags(write=False)
    return m


def sources(name: str, n: int | None = None) -> np.ndarray:
    c = CONFIGS[name]
    if name == "c1":
        src = np.array([[4, 16]], np.int32)
    elif name == "c2":
        src = S.lattice_sources(97, 159, 2)          # 32 x 32 = 1024, walls >= 96 px away
    else:
        src = S.sample_sources(mask(name), c.n_sources, SOURCE_SEED[name])
    return src if n is None else src[:n]
