"""CPU oracle for the FL round loop — TEST INFRASTRUCTURE ONLY.

A plain numpy restatement of the reference algorithm for the hot path
(pkg/src/fedsim: backends/numpy_backend.py, model.py, client.py,
selection.py, server.py; file:line cited per function). It exists to
check the CUDA path, never to run it: only tests/, __graft_entry__.smoke()
and bench.py's cpu_baseline / --impl reference leg may import it. The
product package never imports this directory and has no CPU fallback.

Pinning: tests/test_oracle_golden.py checks this oracle against golden
vectors generated from the reference itself (tests/golden/, made by
tests/golden/make_golden.py importing /root/reference in the build
container): per-kernel outputs, train_local results, per-round aligned
counts and the replay digests of whole runs.
"""
