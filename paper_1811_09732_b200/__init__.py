"""B200-native TrIMS model store (arXiv 1811.09732), load-and-serve hot path.

Native library: ``libtrims.so`` (C++ host + sm_100a CUDA, include/trims.h).
This package is the host-side mirror of the reference's client/daemon API.
"""
from . import format  # noqa: F401
from ._lib import Errc, TrimsError, lib  # noqa: F401
from .format import ModelKey  # noqa: F401

__all__ = ["format", "ModelKey", "TrimsError", "Errc", "lib"]
