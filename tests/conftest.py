"""Shared pytest setup. `-m gpu` tests need a CUDA device and the built
library; `-m "not gpu"` tests run on CPU (oracle pinning, ABI, host logic,
gloo multi-process)."""
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and the built sm_100a library")
    config.addinivalue_line("markers", "slow: long-running")


def fnv1a64(data: bytes) -> str:
    """FNV-1a 64 over raw bytes (the SURVEY's array hash)."""
    h = 0xcbf29ce484222325
    for b in data:
        h ^= b
        h = (h * 0x100000001b3) & 0xFFFFFFFFFFFFFFFF
    return f"{h:016x}"
