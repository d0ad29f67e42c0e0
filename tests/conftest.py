"""Shared pytest configuration.

Markers: ``gpu`` — needs a CUDA device (run on the B200 box with ``-m gpu``).
The repo root is put on sys.path so ``oracle`` (test infrastructure) and the
product package import without installation.
"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")
    config.addinivalue_line("markers", "slow: long-running")
