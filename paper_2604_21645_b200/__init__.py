"""B200-native (sm_100a) PQ / IVF hot path of arxiv/paper_2604_21645 (reference `pqii`).

The compute lives in ``libpqg.so`` (``csrc/``, C ABI in ``include/pqg.h``);
``pqii`` re-exposes the reference's C++ API names over it and ``dist`` shards
rows across GPUs.  Importing the package does not touch the GPU; the first
call loads the library and fails loudly if it is missing.
"""
from . import datagen  # noqa: F401

import importlib as _importlib

__all__ = ["datagen", "pqii", "dist"]


def __getattr__(name):
    if name in ("pqii", "dist"):
        return _importlib.import_module(f"{__name__}.{name}")
    raise AttributeError(name)
