"""Generate golden fixtures from the REFERENCE implementation.

Runs only in the build container (needs /root/reference). It copies the
reference package to a temp dir, builds its Cython backend with the
package's own setup.py (`build_ext --inplace`), imports it under the name
``fedsim_ref`` and records outputs of the reference's own public API:

  rng.npz       derive_seed / shuffle permutations / dropout masks
  kernels.npz   backend forward / loss_and_grad / sign_align_count cases
  train.npz     train_local results (dropout, partial batches, stop/resume)
  agg.npz       aggregate() cases (incl. byte-order ties)
  worlds.json   digests of build_world() outputs for the parity configs
  runs.json     replay digests, per-round aligned counts, reports and
                final-parameter digests of whole FederationEngine runs
  runs_wg.npz   final global parameters of those runs

Usage:  python tests/golden/make_golden.py
"""

from __future__ import annotations

import hashlib
import json
import os
import shutil
import subprocess
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg"


def build_reference() -> str:
    tmp = tempfile.mkdtemp(prefix="fedsim_ref_")
    src = os.path.join(tmp, "pkg")
    shutil.copytree(REF, src)
    for root, dirs, files in os.walk(src):
        os.chmod(root, 0o755)
        for f in files:
            os.chmod(os.path.join(root, f), 0o644)
    subprocess.run([sys.executable, "setup.py", "build_ext", "--inplace"], cwd=src, check=True,
                   stdout=subprocess.DEVNULL)
    pkgroot = os.path.join(tmp, "importroot")
    os.makedirs(pkgroot)
    shutil.copytree(os.path.join(src, "src", "fedsim"), os.path.join(pkgroot, "fedsim_ref"))
    return pkgroot


def world_digest(world, initial) -> str:
    h = hashlib.blake2b(digest_size=8)
    h.update(initial.values.tobytes())
    h.update(np.ascontiguousarray(world.test_features).tobytes())
    h.update(np.ascontiguousarray(world.test_labels).tobytes())
    for wc in world.clients:
        h.update(np.ascontiguousarray(wc.features).tobytes())
        h.update(np.ascontiguousarray(wc.labels).tobytes())
        p = wc.profile
        h.update(repr((p.id, p.speed, p.up_latency_s, p.down_latency_s, p.capacity, wc.batch_size,
                       wc.base_span_s, list(wc.ckpt_capture_offsets))).encode())
    if world.fail_matrix is not None:
        h.update(world.fail_matrix.tobytes())
        h.update(world.fail_offsets.tobytes())
    return h.hexdigest()


PROF = {
    "speed": {"distribution": "loguniform", "low": 20.0, "high": 200.0},
    "capacity": {"distribution": "loguniform", "low": 0.25, "high": 4.0},
    "up_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
    "down_latency": {"distribution": "lognormal", "mu": 0.0, "sigma": 0.5},
}

# Small configs the reference finishes in seconds; every hot-path branch.
RUN_CONFIGS = {
    "sync_weight": {"num_clients": 6, "rounds": 3, "epochs": 2, "dataset": {"n": 1500, "d": 12},
                    "model": {"hidden_dims": [16, 8], "dropout_rate": 0.3}, "seed": 3},
    "sync_delta_dyn": {"num_clients": 8, "rounds": 3, "epochs": 2, "dataset": {"n": 2400, "d": 10},
                       "model": {"hidden_dims": [24, 12], "dropout_rate": 0.3}, "selection_mode": "delta_sign",
                       "batch": {"policy": "dynamic", "b_ref": 16, "b_min": 8, "b_max": 64},
                       "profiles": PROF, "seed": 5},
    "sync_baseline": {"num_clients": 5, "rounds": 2, "epochs": 1, "mode": "sync_baseline",
                      "dataset": {"n": 1200, "d": 9}, "model": {"hidden_dims": [7], "dropout_rate": 0.0},
                      "batch": {"size": 32}, "seed": 11},
    "sync_fail_ckpt": {"num_clients": 6, "rounds": 3, "epochs": 2, "dataset": {"n": 1500, "d": 8},
                       "model": {"hidden_dims": [12, 6], "dropout_rate": 0.3}, "dropout_rate": 0.3,
                       "checkpoint": {"enabled": True, "total_time_s": 60.0, "recovery_s": 2.0},
                       "selection_mode": "delta_sign", "profiles": PROF, "seed": 7},
    "async_fail_lost": {"num_clients": 5, "rounds": 3, "epochs": 1, "mode": "async_filtered",
                        "dataset": {"n": 800, "d": 6}, "model": {"hidden_dims": [5], "dropout_rate": 0.0},
                        "dropout_rate": 0.4, "profiles": PROF, "seed": 13},
    "async_weight": {"num_clients": 6, "rounds": 3, "epochs": 2, "mode": "async_filtered",
                     "dataset": {"n": 1500, "d": 12}, "model": {"hidden_dims": [16, 8], "dropout_rate": 0.3},
                     "profiles": PROF, "seed": 17},
    "async_delta_dyn": {"num_clients": 10, "rounds": 3, "epochs": 2, "mode": "async_filtered",
                        "dataset": {"n": 3000, "d": 10}, "model": {"hidden_dims": [20, 10], "dropout_rate": 0.3},
                        "selection_mode": "delta_sign", "batch": {"policy": "dynamic", "b_ref": 16, "b_min": 8,
                                                                  "b_max": 64},
                        "profiles": PROF, "dropout_rate": 0.1, "checkpoint": {"enabled": True,
                                                                                "total_time_s": 60.0},
                        "seed": 19},
    "unsw_sync_delta": {"num_clients": 16, "rounds": 2, "epochs": 1, "dataset": {"n": 12000, "d": 42},
                        "model": {"hidden_dims": [256, 128, 64], "dropout_rate": 0.3},
                        "selection_mode": "delta_sign", "batch": {"policy": "dynamic"}, "profiles": PROF,
                        "seed": 1},
}


def main() -> None:
    sys.path.insert(0, build_reference())
    os.environ["FEDSIM_BACKEND"] = "compiled"
    import fedsim_ref  # noqa: F401
    from fedsim_ref.backends import _core as core
    from fedsim_ref.client import ClientProfile, train_local
    from fedsim_ref.config import ExperimentConfig
    from fedsim_ref.experiment import build_world
    from fedsim_ref.model import ModelSpec, ParamVector, dropout_masks, init_params
    from fedsim_ref.rng import derive_rng, derive_seed
    from fedsim_ref.server import FederationEngine, aggregate
    import fedsim_ref.selection as sel

    rng = np.random.default_rng(2025)

    # ---------------------------------------------------------------- rng
    masters = [0, 1, 7, 2**31 + 5, 2**40 + 3, 2**63 + 11]
    seeds = []
    for m in masters:
        for cid in (0, 1, 255, 1023):
            for cyc in (0, 3, 49):
                seeds.append((m, cid, cyc, derive_seed(m, "train", cid, cyc)))
    perm_cases = []
    for ts in (1, 12345, 2**62 + 9):
        for n in (1, 2, 7, 171, 1000, 1659):
            for e in (0, 4):
                perm_cases.append((ts, e, n, derive_rng(ts, "shuffle", e).permutation(n)))
    spec = ModelSpec(input_dim=42, hidden_dims=(256, 128, 64), dropout_rate=0.3)
    mask_cases = []
    for ts in (5, 2**50 + 1):
        for (e, s, b) in ((0, 0, 64), (3, 7, 17), (1, 2, 256)):
            ms = derive_seed(ts, "mask", e, s)
            mm = dropout_masks(spec, b, ms)
            mask_cases.append((ts, e, s, b, ms, np.concatenate([x.ravel() for x in mm]) > 0))
    np.savez_compressed(
        os.path.join(HERE, "rng.npz"),
        train_seeds=np.array([s[:3] for s in seeds], dtype=np.uint64),
        train_seed_out=np.array([s[3] for s in seeds], dtype=np.uint64),
        perm_meta=np.array([p[:3] for p in perm_cases], dtype=np.uint64),
        perm_flat=np.concatenate([p[3] for p in perm_cases]).astype(np.int32),
        mask_meta=np.array([m[:5] for m in mask_cases], dtype=np.uint64),
        mask_bits=np.concatenate([np.packbits(m[5], bitorder="little") for m in mask_cases]),
    )

    # ---------------------------------------------------------------- kernels
    kc = {}
    for t in range(24):
        with_masks = t % 2 == 1
        depth = int(rng.integers(1, 4))
        hidden = tuple(int(rng.integers(1, 40)) for _ in range(depth))
        sp = ModelSpec(input_dim=int(rng.integers(1, 30)), hidden_dims=hidden,
                       dropout_rate=0.3 if with_masks else 0.0)
        params = init_params(sp, seed=int(rng.integers(1 << 30)))
        n = int(rng.integers(1, 70))
        x = np.ascontiguousarray(rng.normal(size=(n, sp.input_dim)))
        y = rng.integers(0, 2, n).astype(np.float64)
        mseed = int(rng.integers(1 << 30))
        masks = dropout_masks(sp, n, mseed) if with_masks else None
        loss, grad = core.loss_and_grad(params.values, sp.dims, x, y, masks)
        fwd = core.forward(params.values, sp.dims, x, masks)
        kc[f"c{t}_dims"] = np.array(sp.dims)
        kc[f"c{t}_rate"] = np.array(sp.dropout_rate)
        kc[f"c{t}_w"] = params.values
        kc[f"c{t}_x"] = x
        kc[f"c{t}_y"] = y
        kc[f"c{t}_mseed"] = np.array(mseed if with_masks else -1)
        kc[f"c{t}_loss"] = np.array(loss)
        kc[f"c{t}_grad"] = grad
        kc[f"c{t}_fwd"] = fwd
    for t in range(12):
        n = int(rng.integers(1, 5000))
        a = np.round(rng.normal(size=n), 1)
        b = np.round(rng.normal(size=n), 1)
        a[rng.random(n) < 0.05] = -0.0
        kc[f"s{t}_a"], kc[f"s{t}_b"] = a, b
        kc[f"s{t}_count"] = np.array(core.sign_align_count(a, b))
    np.savez_compressed(os.path.join(HERE, "kernels.npz"), **kc)

    # ---------------------------------------------------------------- train_local
    tr = {}
    prof = ClientProfile(id=0, speed=50.0, up_latency_s=1.0, down_latency_s=1.0, capacity=1.0)
    cases = [((12, (16, 8), 0.3), 40, 3, 16), ((42, (256, 128, 64), 0.3), 171, 2, 64),
             ((9, (7,), 0.0), 25, 2, 8), ((42, (256, 128, 64), 0.3), 300, 1, 256)]
    for t, ((d, hid, rate), n, ep, bs) in enumerate(cases):
        sp = ModelSpec(input_dim=d, hidden_dims=hid, dropout_rate=rate)
        w0 = init_params(sp, 100 + t)
        x = rng.normal(size=(n, d))
        y = rng.integers(0, 2, n).astype(np.int8)
        seed = int(rng.integers(1 << 40))
        upd = train_local(sp, prof, w0, x, y, ep, bs, lambda e: 0.05 * (0.9 ** e), seed)
        tr[f"t{t}_dims"] = np.array(sp.dims)
        tr[f"t{t}_rate"] = np.array(rate)
        tr[f"t{t}_w0"], tr[f"t{t}_x"], tr[f"t{t}_y"] = w0.values, x, y
        tr[f"t{t}_meta"] = np.array([ep, bs, seed], dtype=np.uint64)
        tr[f"t{t}_out"] = upd.params.values
        tr[f"t{t}_steps"] = np.array(upd.steps)
    np.savez_compressed(os.path.join(HERE, "train.npz"), **tr)

    # ---------------------------------------------------------------- aggregate
    ag = {}
    for t in range(10):
        k = int(rng.integers(1, 40))
        m = int(rng.integers(1, 400))
        vecs = [rng.normal(size=m) for _ in range(k)]
        if t % 3 == 0 and k > 2:  # shared leading elements exercise deep byte-order ties
            for v in vecs[1:]:
                v[: min(5, m)] = vecs[0][: min(5, m)]
        out = aggregate([ParamVector(v, "d") for v in vecs])
        ag[f"a{t}_in"] = np.stack(vecs)
        ag[f"a{t}_out"] = out.values
    np.savez_compressed(os.path.join(HERE, "agg.npz"), **ag)

    # ---------------------------------------------------------------- worlds + runs
    worlds, runs, wg = {}, {}, {}
    for name, cfg in RUN_CONFIGS.items():
        conf = ExperimentConfig.from_dict(cfg)
        world, initial = build_world(conf)
        worlds[name] = world_digest(world, initial)
        aligned = []
        orig = sel.calculate_relevance

        def spy(w_c, w_g, w_g_prev=None, mode="weight_sign"):
            score = orig(w_c, w_g, w_g_prev, mode)
            aligned.append(int(score.aligned))
            return score

        sel.calculate_relevance = spy
        try:
            eng = FederationEngine(world)
            state = eng.run(initial)
        finally:
            sel.calculate_relevance = orig
        runs[name] = {
            "config": cfg,
            "digest": eng.timeline.digest(),
            "events": len(eng.timeline.log),
            "aligned": aligned,
            "reports": [r.to_record() for r in eng.reports],
            "params_digest": hashlib.blake2b(state.w_g.values.tobytes(), digest_size=8).hexdigest(),
        }
        wg[name] = state.w_g.values
        print(name, runs[name]["digest"], runs[name]["events"], "events", len(aligned), "scored")
    with open(os.path.join(HERE, "worlds.json"), "w") as f:
        json.dump(worlds, f, indent=1, sort_keys=True)
    with open(os.path.join(HERE, "runs.json"), "w") as f:
        json.dump(runs, f, indent=1, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "runs_wg.npz"), **wg)


if __name__ == "__main__":
    main()
