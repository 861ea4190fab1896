"""GPU simulator (offline window-search inner loop) against the reference's own
outputs (tests/golden sim_* cases).  sim_relu is one CUDA kernel that regenerates the split
randomness from the numpy generator state on the device: bit-exact.  The float pipeline runs in
float64 on the GPU with a different summation order than numpy's im2col matmul: logits within
1e-9 relative, ReLU masks and activation ranges exact on these inputs."""

import numpy as np
import pytest
import torch

import golden_cases as gc
from paper_2309_04875_b200 import models, nn, simulator
from paper_2309_04875_b200.ring import BitWindow, FixedPointConfig

pytestmark = pytest.mark.gpu


def _desk(arch, arrays):
    m = models.desk_cnn(11) if arch == "cnn" else models.desk_mlp(11)
    for k, v in gc.model_weights(arrays, arch).items():
        assert np.array_equal(m.weights[k], v), k
    return m


@pytest.mark.parametrize("case", gc.SIM_RELU_CASES, ids=[c["name"] for c in gc.SIM_RELU_CASES])
def test_sim_relu_bit_exact(golden, case):
    meta, arrays = golden
    rng = np.random.default_rng(np.random.SeedSequence(case["split_seed"]))
    out = simulator.sim_relu(gc.sim_relu_input(case), BitWindow(case["k"], case["m"]), FixedPointConfig(), rng)
    assert np.array_equal(out.view(np.uint64), arrays[case["name"] + "/out"].view(np.uint64))
    # the generator advanced exactly as rng.bytes(8 n) would
    ref = np.random.default_rng(np.random.SeedSequence(case["split_seed"]))
    ref.bytes(8 * case["n"])
    assert rng.bytes(8) == ref.bytes(8)


@pytest.mark.parametrize("mc", gc.SIM_MODEL_CASES, ids=[c["name"] for c in gc.SIM_MODEL_CASES])
def test_sim_forward_vs_reference(golden, mc):
    meta, arrays = golden
    g = meta[mc["name"]]
    model = _desk(mc["arch"], arrays)
    x_f, labels = gc.sim_model_inputs(mc)
    cfg = simulator.SimConfig(FixedPointConfig(), [None if w is None else BitWindow(*w) for w in mc["windows"]],
                              seed=mc["seed"])
    logits, acc = simulator.sim_forward(model, x_f, labels, cfg)
    np.testing.assert_allclose(logits, arrays[mc["name"] + "/logits"], rtol=1e-9, atol=1e-12)
    assert acc == g["accuracy"]
    _, masks = simulator.collect_drelu_decisions(model, x_f, cfg)
    assert len(masks) == g["n_masks"]
    for i, mk in enumerate(masks):
        assert np.array_equal(mk, arrays[mc["name"] + f"/mask{i}"])
    np.testing.assert_allclose(simulator.plain_forward(model, x_f), arrays[mc["name"] + "/plain"], rtol=1e-9,
                               atol=1e-12)
    assert {str(k): v for k, v in simulator.collect_activation_ranges(model, x_f).items()} == g["ranges"]


def test_sim_forward_resnet18_runs():
    """The simulator on a model the reference cannot express (ResNet18-CIFAR, Residual blocks):
    the windowed forward tracks the exact forward, and a wider window tracks it more closely."""
    model = models.resnet18_cifar(0)
    x_f = np.random.default_rng(2).uniform(0, 1, (4, 3, 32, 32))
    plain = simulator.plain_forward(model, x_f)
    errs = []
    for k, m in ((40, 0), (22, 10)):
        cfg = simulator.SimConfig(FixedPointConfig(), [BitWindow(k, m)] * model.n_groups, seed=1)
        logits, _ = simulator.sim_forward(model, x_f, None, cfg)
        assert logits.shape == (4, 10) and np.all(np.isfinite(logits))
        errs.append(np.max(np.abs(logits - plain)))
    assert errs[0] <= errs[1] + 1e-12 and errs[0] < 1e-6
    ranges = simulator.collect_activation_ranges(model, x_f)
    assert set(ranges) == set(range(model.n_groups)) and all(2 <= v <= 64 for v in ranges.values())
    _ = torch


@pytest.mark.parametrize("case", gc.SEARCH_CASES, ids=[c["name"] for c in gc.SEARCH_CASES])
def test_window_search_vs_reference(golden, case):
    """search_eco / search_budget over the GPU simulator return the reference's windows, accuracy,
    baseline, bit fraction and search trace (tests/golden/golden_search.json, made by running the
    reference search on its desk CNN)."""
    import json
    import os

    from paper_2309_04875_b200 import search

    with open(os.path.join(os.path.dirname(__file__), "golden", "golden_search.json")) as fh:
        want = json.load(fh)[case["name"]]
    model = _desk("cnn", golden[1])
    x_f, labels = gc.search_inputs(case)
    if case["kind"] == "eco":
        res = search.search_eco(model, x_f, labels, seed=case["seed"])
    else:
        res = search.search_budget(model, x_f, labels, case["budget"], threshold=case.get("threshold"),
                                   candidate_widths=tuple(case["widths"]), seed=case["seed"])
    assert res.to_json() == want
