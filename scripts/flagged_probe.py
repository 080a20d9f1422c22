"""Flagged K3 probe (diagnostic): the step-published keep bits alone vs the
plan's complete bits, then K3-before-trainer and trainer-before-K3."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2503_15448_b200 import device as D  # noqa: E402
from paper_2503_15448_b200.model import ModelSpec, init_params  # noqa: E402

spec = ModelSpec(input_dim=42, hidden_dims=(256, 128, 64), dropout_rate=0.3)
rng = np.random.default_rng(3)
sizes = [300, 77, 1024, 64, 500, 129]
feats = [rng.normal(size=(n, 42)) for n in sizes]
labs = [(rng.random(n) < 0.3).astype(np.int8) for n in sizes]
rt = D.Runtime.get()
shards = D.DeviceShards(feats, labs, rt)
w0 = torch.tensor(init_params(spec, 5).values, dtype=torch.float32, device="cuda")
k = len(sizes)
clients, seeds = np.arange(k), np.arange(k, dtype=np.uint64) + 40
batch = np.array([64, 64, 128, 64, 256, 64])
lr = np.full((k, 5), 0.05)
starts = np.full(k, w0.data_ptr(), dtype=np.uint64)
ref = D.TrainPlan(spec.dims, shards, clients, seeds, batch, 5, 0.3, rt=rt)
want, st_want = D.run_trainer(ref, lr, starts, "bf16")
torch.cuda.synchronize()


def flagged(plan, flags, stream):
    rt.call(rt.lib.fs_dropout_bits_flagged(plan.seeds_p, plan.n_rows_p, plan.batch_p, plan.mask_off_p,
                                           plan.order_p, k, 5, plan.max_steps, plan.sum_hidden, 0.7,
                                           plan.bits.data_ptr(), flags.data_ptr(), 7, stream.cuda_stream),
            "fs_dropout_bits_flagged")


plan = D.TrainPlan(spec.dims, shards, clients, seeds, batch, 5, 0.3, rt=rt)
torch.cuda.synchronize()
plan.bits.zero_()
flags = torch.zeros(k * plan.max_steps, dtype=torch.int32, device="cuda")
flagged(plan, flags, torch.cuda.current_stream())
torch.cuda.synchronize()
print("max_steps", plan.max_steps, "flags set", int((flags == 7).sum()), "of", flags.numel())
print("bits equal", torch.equal(plan.bits, ref.bits), "nonzero ref", int((ref.bits != 0).sum()),
      "nonzero got", int((plan.bits != 0).sum()), "diff words", int((plan.bits != ref.bits).sum()))
sys.stdout.flush()
# K3 first, then the trainer waiting on flags
plan2 = D.TrainPlan(spec.dims, shards, clients, seeds, batch, 5, 0.3, rt=rt)
torch.cuda.synchronize()
plan2.bits.zero_()
flags2 = torch.zeros(k * plan2.max_steps, dtype=torch.int32, device="cuda")
plan2.mask_flags, plan2.mask_tag = flags2, 7
side = torch.cuda.Stream()
side.wait_stream(torch.cuda.current_stream())
flagged(plan2, flags2, side)
got, st = D.run_trainer(plan2, lr, starts, "bf16")
torch.cuda.synchronize()
print("K3 first: rows equal", torch.equal(got, want), "status", st.tolist())
sys.stdout.flush()
# trainer first on a non-default stream, K3 after it on another
plan3 = D.TrainPlan(spec.dims, shards, clients, seeds, batch, 5, 0.3, rt=rt)
torch.cuda.synchronize()
plan3.bits.zero_()
flags3 = torch.zeros(k * plan3.max_steps, dtype=torch.int32, device="cuda")
plan3.mask_flags, plan3.mask_tag = flags3, 7
main, side = torch.cuda.Stream(), torch.cuda.Stream()
main.wait_stream(torch.cuda.current_stream())
side.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(main):
    got, st = D.run_trainer(plan3, lr, starts, "bf16")
flagged(plan3, flags3, side)
torch.cuda.synchronize()
print("trainer first: rows equal", torch.equal(got, want), "status", st.tolist())
