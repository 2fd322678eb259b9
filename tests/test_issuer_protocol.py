"""The attention kernel's warp-role protocol (MMA issuer, K/V/Q/key-coordinate rings, softmax
pv_done bookkeeping) is deadlock-free and never aliases an mbarrier phase, over random per-half
tile-liveness patterns and ring depths (tests/issuer_sim.py mirrors csrc/attn.cu)."""
import random

import pytest

import issuer_sim


@pytest.mark.parametrize("kst", [2, 3])
@pytest.mark.parametrize("issuer", ["static", "static-s64", "dynamic"])
def test_issuer_protocol_random(kst, issuer):
    rnd = random.Random(100 + kst)
    for trial in range(200):
        items = issuer_sim.rand_items(rnd, rnd.randint(1, 6))
        r, state, alive = issuer_sim.run(items, KST=kst, VST=kst, seed=trial, issuer=issuer.split("-")[0],
                                         s64=issuer.endswith("s64"))
        assert r == "ok", (trial, items, alive, state)


def test_issuer_protocol_detects_coupled_order():
    """The model is sharp: the first dynamic issuer (P(t, 1) V queued behind S(t', 0), which waits
    for a K load) deadlocks on this liveness pattern, and the model finds it."""
    items = [dict(n=9, has_b=True, live=[3, 1, 3, 2, 2, 2, 2, 3, 3], kp=[True, True, True, True, False, True, False, False, True])]
    found = False
    for seed in range(200):
        r, _, _ = issuer_sim.run(items, seed=seed, issuer="dynamic", coupled=True)
        if r != "ok":
            found = True
            break
    assert found
