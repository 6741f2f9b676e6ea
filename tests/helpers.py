"""Shared test helpers (mirrors the reference tests' rand_vec / relerr,
reference tests/test_hankel.py:8-13)."""

import os

import numpy as np

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def rand_vec(rng, n):
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def relerr(a, b):
    """Reference test metric ||a-b|| / (||b|| + 1)."""
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (np.linalg.norm(b) + 1.0)


def strict_relerr(a, b):
    """SURVEY §7 parity metric ||a-b|| / ||b|| (stricter than the +1 form)."""
    nb = np.linalg.norm(b)
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / (nb if nb > 0 else 1.0)


def load_small_cases():
    return np.load(os.path.join(GOLDEN, "small_cases.npy"), allow_pickle=True).item()


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)
