"""Acceptance criterion 7 (acceptance_main.cpp:278-335) on the device path:
oscar < rotate-only < kivi and scale-only > kivi in >= 18 of 20 seeds, with
the output MSE of simulate_fidelity (pipeline.cpp:359-408) measured through
the CUDA cache (paper_2605_19660_b200/fidelity.py)."""
import json
import os

import pytest

pytestmark = pytest.mark.gpu


def test_method_ordering_on_device():
    from paper_2605_19660_b200 import fidelity as fd

    cnt = fd.method_ordering(seeds=range(1, 21))
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "gpurun_out")
    if os.path.isdir(d):
        with open(os.path.join(d, "fidelity_ordering.json"), "w") as f:
            json.dump(cnt, f)
    assert cnt["oscar<rotate-only"] >= 18, cnt
    assert cnt["rotate-only<kivi"] >= 18, cnt
    assert cnt["scale-only>kivi"] >= 18, cnt
