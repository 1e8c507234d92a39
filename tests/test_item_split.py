"""K4 work-item sizing: head items and the tail re-cut into smaller items
(guided self-scheduling, glsim_cuda.cu plan_items) must not change any
result.  Small designs only reach the coarse-item and tail paths when the
sizing assumes few workers (gs_engine_set_items via simcore.ENGINE_ITEMS);
every setting is checked against the oracle."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pct", [100, 50])
def test_item_split_matches_oracle(oracle_lib, pct):
    from test_full_size_parity import _oracle_stats
    import paper_2203_06117_b200 as api
    from paper_2203_06117_b200 import simcore, synth
    cfg = synth.config("C2", gates=3000, windows=3000)
    m = synth.design(cfg)
    stim = synth.stimulus(cfg, 0, 3000)
    ref, a = _oracle_stats(oracle_lib, m, stim, pct)
    settings = [None,          # grid-sized items
                (16, 1, 2),    # coarse items, no tail
                (16, 2, 2),    # coarse head + tail
                (64, 4, 1),    # finer tail, always re-cut
                (1, 2, 2)]     # one worker: the largest items
    try:
        for items in settings:
            simcore.ENGINE_ITEMS = items
            stats, diag = api.simulate_streaming(m, stim, api.RunConfig(pathpulse_pct=pct))
            for f in ("t0", "t1", "tc", "ig"):
                assert np.array_equal(getattr(stats, f), ref[f]), f"{items} {f}"
            assert diag["discarded"] == int(a["discarded"].sum()), items
            assert diag["ic_filtered"] == int(a["ic_filtered"].sum()), items
    finally:
        simcore.ENGINE_ITEMS = None


def test_item_sizing_rejects_bad_values():
    from paper_2203_06117_b200 import _native, synth
    m = synth.design(synth.config("C2", gates=1000, levels=2))
    eng = _native.Engine(m.device(), 0)
    for bad in ((-1, 2, 2), (0, 0, 2), (0, 2, 0)):
        with pytest.raises(ValueError):
            eng.set_items(*bad)
