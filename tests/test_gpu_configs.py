"""Parity against the REFERENCE at the BASELINE.json configurations.

Fixtures (tests/golden/configs.json + configs_wg.npz) were recorded from the
reference package itself (tests/golden/make_golden_configs.py): C1 (10
UNSW-shaped clients, 5 rounds, sync_baseline), C2 (100 clients,
async_filtered, dynamic batch, delta_sign, 2 windows), C3 (256 ROAD-shaped
clients, sync_filtered, 2 rounds) and C4 (1024 clients, sync_filtered,
dynamic batch, delta_sign, 5 rounds, with the global model after every
round).

fp64 parity mode (first row): identical replay digest,
identical per-round aligned counts of every scored client, reports'
accuracy/AUC within 1e-9 and the global model within 1e-12 relative.

bf16 mode (second row), C4, teacher-forced on the
reference's own model sequence: round r (1..4) is run from the reference's
w_g(r) and w_g(r-1); the selection decisions must equal the reference's for
every client whose reference ratio is more than EPS_R = 5e-3 from theta
(flips inside the band and the band occupancy are reported, not hidden);
the teacher-forced next model and a free-running 5-round bf16 run must stay
within the stated relative-L2 bounds of the reference's models, and the
free run's accuracy/AUC within 0.5 points of the reference's.
"""

from __future__ import annotations

import json
import os

import numpy as np
import pytest

from tests.conftest import GOLDEN, cuda_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not cuda_ok(), reason="needs a CUDA device")]

EPS_R = 5e-3            # near-threshold band |aligned_ref/M - theta| <= EPS_R
TF_WG_REL_L2 = 2e-3     # teacher-forced w_g(r+1): ||w_bf16 - w_ref|| / ||w_ref||
FREE_WG_REL_L2 = 1e-2   # free-running 5-round bf16 w_g vs the reference's
QUALITY_PTS = 0.005     # accuracy and AUC within 0.5 points


@pytest.fixture(scope="module")
def configs():
    with open(os.path.join(GOLDEN, "configs.json")) as f:
        recs = json.load(f)
    return recs, dict(np.load(os.path.join(GOLDEN, "configs_wg.npz")))


def _world(cfg, precision):
    from paper_2503_15448_b200.config import ExperimentConfig
    from paper_2503_15448_b200.experiment import build_world

    return build_world(ExperimentConfig.from_dict(cfg), precision=precision)


def _aligned_by_round(log, M):
    out = {}
    for rec in log:
        if rec["kind"] == "train_done" and rec.get("relevance") is not None:
            out.setdefault(str(rec["round"]), []).append((rec["client_id"], int(round(rec["relevance"] * M))))
    return {r: [a for _, a in sorted(v)] for r, v in out.items()}


def _rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


@pytest.mark.parametrize("name", ["c1_sync", "c2_async", "c3_sync", "c4_sync"])
def test_fp64_engine_replays_reference_at_baseline_config(configs, name):
    from paper_2503_15448_b200.server import FederationEngine

    recs, wg = configs
    ref = recs[name]
    world, initial = _world(ref["config"], "fp64")
    eng = FederationEngine(world)
    state = eng.run(initial)
    log = list(eng.timeline.log)
    assert len(log) == ref["events"]
    assert _aligned_by_round(log, ref["M"]) == ref["aligned"]
    assert eng.timeline.digest() == ref["digest"]
    for mine, theirs in zip(eng.reports, ref["reports"]):
        assert abs(mine.accuracy - theirs["accuracy"]) <= 1e-9 and abs(mine.auc - theirs["auc"]) <= 1e-9
    w_ref = wg[f"{name}_wg"]
    err = float(np.max(np.abs(state.w_g.values - w_ref) / np.maximum(np.abs(w_ref), 1.0)))
    assert err <= 1e-12, err


def test_fp64_c4_round_models_match_reference(configs):
    """Every round's global model of the C4 run, not only the last."""
    from paper_2503_15448_b200.server import FederationEngine, GlobalState

    recs, wg = configs
    models = wg["c4_sync_models"]
    world, initial = _world(recs["c4_sync"]["config"], "fp64")
    eng = FederationEngine(world)
    st = GlobalState(round=0, w_g=initial)
    assert np.array_equal(initial.values, models[0])
    for r in range(1, len(models)):
        st = eng.run_sync_round(st)
        err = float(np.max(np.abs(st.w_g.values - models[r]) / np.maximum(np.abs(models[r]), 1.0)))
        assert err <= 1e-12, (r, err)


def test_bf16_c4_teacher_forced_masks_and_models(configs):
    """Teacher-forced bf16 rounds at the headline shape (1024 clients)."""
    from paper_2503_15448_b200.model import ParamVector
    from paper_2503_15448_b200.server import FederationEngine, GlobalState

    recs, wg = configs
    ref = recs["c4_sync"]
    models = wg["c4_sync_models"]
    M, theta = ref["M"], ref["config"]["theta"]
    world, initial = _world(ref["config"], "bf16")
    digest = initial.spec_digest
    report = []
    for r in range(1, len(models) - 1):
        eng = FederationEngine(world)
        st = GlobalState(round=r, w_g=ParamVector(models[r], digest), w_g_prev=ParamVector(models[r - 1], digest))
        st = eng.run_sync_round(st)
        mine = np.array(_aligned_by_round(list(eng.timeline.log), M)[str(r)]) / M
        theirs = np.array(ref["aligned"][str(r)]) / M
        assert mine.shape == theirs.shape == (world.num_clients,)
        flip = (mine >= theta) != (theirs >= theta)
        band = np.abs(theirs - theta) <= EPS_R
        tf_err = _rel_l2(st.w_g.values, models[r + 1])
        report.append({"round": r, "flips": int(flip.sum()), "flips_outside_band": int((flip & ~band).sum()),
                       "band_occupancy": int(band.sum()), "max_abs_dratio": float(np.max(np.abs(mine - theirs))),
                       "accepted_ref": int((theirs >= theta).sum()), "accepted_bf16": int((mine >= theta).sum()),
                       "wg_rel_l2": tf_err})
    print("bf16 teacher-forced C4:", json.dumps(report))
    for row in report:
        assert row["flips_outside_band"] == 0, row
        assert row["wg_rel_l2"] <= TF_WG_REL_L2, row


def test_bf16_c4_free_run_tracks_reference(configs):
    """Free-running bf16 C4 rounds from the reference's initial model: global
    model and accuracy/AUC after 5 rounds against the reference's."""
    from paper_2503_15448_b200.server import FederationEngine, GlobalState

    recs, wg = configs
    ref = recs["c4_sync"]
    models = wg["c4_sync_models"]
    world, initial = _world(ref["config"], "bf16")
    eng = FederationEngine(world)
    st = GlobalState(round=0, w_g=initial)
    errs = []
    for r in range(1, len(models)):
        st = eng.run_sync_round(st)
        errs.append(_rel_l2(st.w_g.values, models[r]))
    last, ref_last = eng.reports[-1], ref["reports"][-1]
    print("bf16 free-run C4 rel-L2 per round:", errs, "acc", last.accuracy, ref_last["accuracy"],
          "auc", last.auc, ref_last["auc"])
    assert errs[-1] <= FREE_WG_REL_L2, errs
    assert abs(last.accuracy - ref_last["accuracy"]) <= QUALITY_PTS
    assert abs(last.auc - ref_last["auc"]) <= QUALITY_PTS
