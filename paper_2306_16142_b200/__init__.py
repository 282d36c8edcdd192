"""B200-native DDF path-tracing hot path (arXiv 2306.16142), drop-in behind
the reference ``ddfield`` backend protocol and ``render.render_path``.

Importing the package does not touch the GPU; the first field construction
loads ``lib/libddf_b200.so`` and fails loudly without a B200.
"""

from .errors import DataError, DdfError, NumericError  # noqa: F401
from .neural import MlpModel, kaiming_uniform, load_model, save_model  # noqa: F401

__all__ = ["DataError", "DdfError", "NumericError", "MlpModel", "kaiming_uniform", "load_model",
           "save_model"]
