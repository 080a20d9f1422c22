"""Helpers for running the REFERENCE package (oracle/_ref/pkg, built by
oracle/build_ref.sh) as a checker and CPU baseline. Test/bench
infrastructure only: tests/, tests/golden/ scripts and bench.py's reference
arm and cpu_baseline leg import it; the product never does.

``use_reference()`` puts the built reference tree first on sys.path (the
package keeps its own name, ``fedsim``) with its compiled Cython backend.

``ForkPoolExecutor`` stands in for ``concurrent.futures.ThreadPoolExecutor``
inside the reference's ``run_sync_round`` (pkg/src/fedsim/server.py:412-415):
the reference fans a round's clients out over a thread pool when
``world.workers > 1``, but its client loop holds the GIL (a thread pool over 8
cores was measured slower than one thread). Forked worker
processes give the reference's own code path every host core: ``map(fn,
items)`` forks the workers (fn and everything it closes over -- world,
w_g, w_g_prev -- are inherited), evaluates fn on the items and returns the
results in item order, exactly what the thread pool's ``map`` returns.
Every client cycle is a pure function of its inputs (server.py:196-301), so
the event log and model are identical to the serial run's.
"""

from __future__ import annotations

import multiprocessing as mp
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
REF_SRC = os.path.join(HERE, "_ref", "pkg", "src")


def use_reference(backend: str = "compiled"):
    """Import the built reference package (raises if oracle/_ref is missing)."""
    if not os.path.isdir(os.path.join(REF_SRC, "fedsim")):
        raise ImportError("oracle/_ref/pkg not built (run oracle/build_ref.sh where /root/reference exists)")
    os.environ["FEDSIM_BACKEND"] = backend
    os.environ.setdefault("OPENBLAS_NUM_THREADS", "1")
    if REF_SRC not in sys.path:
        sys.path.insert(0, REF_SRC)
    import fedsim

    if not os.path.abspath(fedsim.__file__).startswith(REF_SRC):
        raise ImportError(f"a different fedsim package is on the path: {fedsim.__file__}")
    return fedsim


class ForkPoolExecutor:
    """ThreadPoolExecutor stand-in whose map() runs in forked processes."""

    _fn = None

    def __init__(self, max_workers: int | None = None):
        self.n = max(1, int(max_workers or os.cpu_count() or 1))

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        return False

    def map(self, fn, items):
        items = list(items)
        if self.n == 1 or len(items) <= 1:
            return [fn(i) for i in items]
        ForkPoolExecutor._fn = fn
        try:
            with mp.get_context("fork").Pool(min(self.n, len(items))) as pool:
                # small chunks: client costs are ragged (n_i from 1 to ~1.7k rows)
                return pool.map(_call, items, chunksize=max(1, len(items) // (16 * self.n)))
        finally:
            ForkPoolExecutor._fn = None


def _call(item):
    return ForkPoolExecutor._fn(item)


def patch_server_pool(server_module) -> None:
    """Route the reference server's client fan-out through ForkPoolExecutor."""
    server_module.ThreadPoolExecutor = ForkPoolExecutor
