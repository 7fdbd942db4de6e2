"""B200-native low-rank NUFFT (arXiv:1701.04492): sm_100a kernels behind the
reference's NUFFT-I/II/III/2D entry points.  See DESIGN.md."""
from .api import *  # noqa: F401,F403
from .api import __all__ as _api_all
from ._lib import LIB_PATH, exported_symbols, lib  # noqa: F401
from . import parallel  # noqa: F401
from .parallel import NcclComm  # noqa: F401

__all__ = list(_api_all) + ["LIB_PATH", "exported_symbols", "lib", "parallel", "NcclComm"]
