"""fedsim-b200: the FL round loop of arXiv 2503.15448 on sm_100a.

Drop-in for the reference ``fedsim`` package's hot-path API (backends,
model, client, selection, server, simnet) with all per-round arithmetic in
hand-written CUDA kernels behind a C-ABI library (include/fedsim_b200.h).
"""

__version__ = "0.1.0"


def backend_name() -> str:
    from .backends import backend_name as _bn

    return _bn()
