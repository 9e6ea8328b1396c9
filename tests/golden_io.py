"""Helpers to read the committed golden fixtures (tests/golden/*.npz)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def cores(z, prefix):
    d = int(z[f"{prefix}__d"])
    return [np.array(z[f"{prefix}__{k}"]) for k in range(d)]


def factors(z, prefix):
    out, k = [], 0
    while f"{prefix}_F__{k}" in z:
        out.append(np.array(z[f"{prefix}_F__{k}"]))
        k += 1
    return out
