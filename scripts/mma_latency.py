"""tcgen05 stage latency: one thread issues n MMAs (M=128, N, K=16) + commit,
waits on the mbarrier; operands SWIZZLE_NONE core matrices vs 128B swizzle;
the MMAs accumulate into `nacc` independent TMEM accumulators round-robin
(diagnostic for the bf16 trainer's per-stage cost)."""
import ctypes
import os

lib = ctypes.CDLL(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests",
                               "_mma_latency_probe.so"))
lib.probe_mma_latency.restype = ctypes.c_longlong
for n in (64, 128):
    for k in (4, 8, 16):
        for nacc in (1,):
            if n * nacc > 512:
                continue
            row = [lib.probe_mma_latency(s, n, k, nacc, 50) for s in (0, 1, 2, 3, 8, 11)]
            print(f"N={n:3d} mmas={k:2d} acc={nacc} floor={128 * n // 256 * k:5d}  none={row[0]:6d}  sw128={row[1]:6d}  "
                  f"none-incremental={row[2]:6d}  const={row[3]:6d}  | icache thrashed: none={row[4]:6d}  const={row[5]:6d}")
