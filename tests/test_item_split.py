"""K4 work-item sizing: head items of tpi tiles and the tail re-cut into
smaller items (guided self-scheduling, glsim_cuda.cu gs_run K4 loop) must not
change any result.  Small designs only reach those paths when the item sizing
assumes few warps (GS_ITEM_WARPS, read once per process), so each setting runs
in its own subprocess; every one is checked against the oracle."""

import json
import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r"""
import json, sys
import numpy as np
sys.path.insert(0, sys.argv[1])
import paper_2203_06117_b200 as api
from paper_2203_06117_b200 import synth
cfg = synth.config("C2", gates=3000, windows=3000)
m = synth.design(cfg)
stim = synth.stimulus(cfg, 0, 3000)
stats, diag = api.simulate_streaming(m, stim, api.RunConfig(pathpulse_pct=int(sys.argv[2])))
print(json.dumps({f: np.asarray(getattr(stats, f)).tolist() for f in ("t0", "t1", "tc", "ig")}
                 | {"ic_filtered": int(diag["ic_filtered"]), "discarded": int(diag["discarded"])}))
"""


def _run(env_extra, pct):
    env = dict(os.environ, **env_extra)
    out = subprocess.run([sys.executable, "-c", CHILD, ROOT, str(pct)], env=env,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    return json.loads(out.stdout.strip().splitlines()[-1])


@pytest.mark.parametrize("pct", [100, 50])
def test_item_split_matches_oracle(oracle_lib, pct):
    from test_full_size_parity import _oracle_stats
    from paper_2203_06117_b200 import synth
    cfg = synth.config("C2", gates=3000, windows=3000)
    m = synth.design(cfg)
    stim = synth.stimulus(cfg, 0, 3000)
    ref, a = _oracle_stats(oracle_lib, m, stim, pct)
    settings = [{},                                              # grid-sized items
                {"GS_ITEM_WARPS": "16", "GS_TAIL_DIV": "1"},      # coarse items, no tail
                {"GS_ITEM_WARPS": "16"},                          # coarse head + tail
                {"GS_ITEM_WARPS": "64", "GS_TAIL_DIV": "4", "GS_TAIL_FRAC": "1"}]
    for env in settings:
        got = _run(env, pct)
        for f in ("t0", "t1", "tc", "ig"):
            assert np.array_equal(np.asarray(got[f]), ref[f]), f"{env} {f}"
        assert got["discarded"] == int(a["discarded"].sum()), env
        assert got["ic_filtered"] == int(a["ic_filtered"].sum()), env
