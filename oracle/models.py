"""Oracle model drivers (ResNet-50-shaped forward, LSTM) -- TEST INFRASTRUCTURE.

Bound lazily from liboracle.so when their C sources are present.
"""
from __future__ import annotations


def register(L) -> None:
    """Declare ctypes signatures for the model-level oracle entry points that exist."""
    return None
