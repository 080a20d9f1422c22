"""Round-time probe for the next round's dropout bits (K3): C4 bf16 rounds
(1) as built, (2) with K3 as the fine-grained one-(client, step)-per-CTA kernel
(short CTAs free SMs for the round's high-priority tail kernels sooner),
(3) without K3 (bit buffers keep an earlier round's bits: timing only)."""
import ctypes
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2503_15448_b200 import device as D  # noqa: E402

world, init = bench.build_c4_world(precision="bf16")
world.device_state()
r = bench.measure_rounds(world, init, None, steps=20, warmup=5, device_index=0)
print("as built        ms/round %.4f  median %.4f" % (r["ms_per_round"], sorted(r["round_ms"])[10]))
eng = r["engine"]
max_steps = max(p.max_steps for p in eng._plans.values())
rt = D.Runtime.get()
lib = rt.lib
n = world.num_clients
order = torch.arange(n, dtype=torch.int32, device="cuda")
flags = torch.zeros(n * 256, dtype=torch.int32, device="cuda")
orig = lib.fs_dropout_bits


def fine(seeds, n_rows, batch, mask_off, n_req, epochs, sum_hidden, keep, bits, stream):
    return lib.fs_dropout_bits_flagged(seeds, n_rows, batch, mask_off, order.data_ptr(), n_req, epochs, 256,
                                       sum_hidden, keep, bits, flags.data_ptr(), 1, stream)


lib.fs_dropout_bits = fine
r = bench.measure_rounds(world, init, None, steps=20, warmup=5, device_index=0)
print("fine-grained K3 ms/round %.4f  median %.4f (max_steps %d)" % (r["ms_per_round"], sorted(r["round_ms"])[10], max_steps))
lib.fs_dropout_bits = lambda *a: 0
r = bench.measure_rounds(world, init, None, steps=20, warmup=5, device_index=0)
print("without K3      ms/round %.4f  median %.4f" % (r["ms_per_round"], sorted(r["round_ms"])[10]))
