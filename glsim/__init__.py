"""``import glsim`` compatibility alias for :mod:`paper_2203_06117_b200`.

Code written against the reference package (``glsim``, including
``glsim.scheduler.simcore.two_pass_simulate`` / ``glsim.simcore.verify_two_pass``
monkeypatch points and ``from glsim.oracle import ...``) runs unchanged: every
``glsim.<module>`` below is the *same module object* as the B200 package's.
"""

import sys

import paper_2203_06117_b200 as _pkg
from paper_2203_06117_b200 import *  # noqa: F401,F403
from paper_2203_06117_b200 import (__all__, __version__, cli, errors, eventsim, netlist,  # noqa
                                   report, scheduler, sdf, simcore, waveform)

oracle = eventsim
for _name, _mod in (("cli", cli), ("errors", errors), ("netlist", netlist),
                    ("oracle", eventsim), ("report", report), ("scheduler", scheduler),
                    ("sdf", sdf), ("simcore", simcore), ("waveform", waveform)):
    sys.modules[f"{__name__}.{_name}"] = _mod
del _name, _mod, _pkg
