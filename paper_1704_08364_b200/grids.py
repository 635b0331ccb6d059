"""``tomoblocks.grids``-compatible import path (see slices.py)."""
from .slices import *  # noqa: F401,F403
from .slices import __all__  # noqa: F401
