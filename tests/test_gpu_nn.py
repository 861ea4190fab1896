"""GPU parity of the ring linear layers and the model-level entry.

Bar: bit-exact.  Layer outputs per party equal the reference's nn.linear_forward /
conv2d_forward / avgpool_forward / truncate_local on the same shares (golden
digests); run_local_forward reproduces the reference's logits SHA, meters and
per-layer logs on its desk models; ResNet-shaped models (residual blocks, which
the reference cannot express) match the oracle share for share.
"""

import numpy as np
import pytest
import torch

import golden_cases as gc
from hb_helpers import sha
from oracle import hb_oracle as O
from oracle import hb_oracle_nn as ON
from paper_2309_04875_b200 import models, nn
from paper_2309_04875_b200.ring import BitWindow, FixedPointConfig
from paper_2309_04875_b200.sharing import ArithShareTensor

pytestmark = pytest.mark.gpu


class _Sess:
    fxp = FixedPointConfig(64, 16)


@pytest.mark.parametrize("case", gc.NN_CASES, ids=[c["name"] for c in gc.NN_CASES])
def test_nn_layer_golden(golden, case):
    g = golden[0][case["name"]]
    ins = gc.make_nn_inputs(case)
    for p in (0, 1):
        x = ArithShareTensor(p, 64, ins[f"x{p}"])
        if case["op"] == "linear":
            y = nn.linear_forward(_Sess, x, ins["w"], ins["b"])
        elif case["op"] == "conv":
            y = nn.conv2d_forward(_Sess, x, nn.Conv2d(*case["layer"], weight="w", bias="b"), ins["w"], ins["b"])
        elif case["op"] == "avgpool":
            y = nn.avgpool_forward(_Sess, x, nn.AvgPool(*case["layer"]))
        else:
            y = nn.truncate_local(x, _Sess.fxp)
        assert list(y.shape) == g["shape"]
        assert sha(y.data) == g[f"y{p}_sha"], (case["name"], p)


def _desk(arch, arrays):
    m = models.desk_cnn(11) if arch == "cnn" else models.desk_mlp(11)
    for k, v in gc.model_weights(arrays, arch).items():  # the reference's own draws
        assert np.array_equal(m.weights[k], v), k
    return m


@pytest.mark.parametrize("pair", [True, False], ids=["pair", "threads"])
@pytest.mark.parametrize("mc", gc.MODEL_CASES, ids=[c["name"] for c in gc.MODEL_CASES])
def test_run_local_forward_golden(golden, mc, pair):
    meta, arrays = golden
    g = meta[mc["name"]]
    model = _desk(mc["arch"], arrays)
    cfg = nn.ReluConfig([None if w is None else BitWindow(*w) for w in mc["windows"]])
    logits, meters, logs, _ = nn.run_local_forward(model, cfg, gc.model_inputs(mc), mc["seed"], pair=pair)
    assert O.digest(np.ascontiguousarray(logits).view(np.uint64)) == g["logits_sha"]
    assert meters[0].to_json() == g["meter0"] and meters[1].to_json() == g["meter1"]
    assert logs[0] == g["layers0"] and logs[1] == g["layers1"]


def _tiny_resnet():
    ini = models._Init(3)
    layers = [ini.conv("stem", 3, 8, 3, 1, 1), nn.Relu(0)]
    layers += models._basic_block(ini, "b1", 8, 8, 1, 1)
    layers += models._basic_block(ini, "b2", 8, 16, 2, 2)
    layers += models._bottleneck(ini, "b3", 16, 4, 1, 2)
    layers += [nn.AvgPool(4, 4, 4), nn.Flatten(), ini.linear("fc", 16, 10)]
    return nn.ModelSpec(FixedPointConfig(), (3, 8, 8), layers, ini.weights)


@pytest.mark.parametrize("windows", [[(22, 14)] * 3, [(64, 0), (20, 6), None]], ids=["w8", "mixed"])
def test_resnet_shaped_vs_oracle(windows):
    model = _tiny_resnet()
    x_f = np.random.default_rng(5).uniform(0, 1, (6, 3, 8, 8))
    cfg = nn.ReluConfig([None if w is None else BitWindow(*w) for w in windows])
    layers = [nn._layer_to_json(L) for L in model.layers]
    want, traces, wlogs = ON.run_local_forward(layers, model.input_shape, model.weights, windows, x_f, 9)
    for pair in (True, False):
        logits, meters, logs, _ = nn.run_local_forward(model, cfg, x_f, 9, pair=pair)
        assert np.array_equal(logits, want)
        assert logs[0] == wlogs[0]
        assert [tuple(t) for t in meters[0].trace] == [tuple(t) for t in traces[0]]


def _wide_resnet():
    """ResNet-shaped, wide enough (>= 64 channels) for the TMA conv kernels: the 3-channel stem on
    the gather kernel, a basic block on k_conv_tma<64,1,..> with the residual add fused into its
    epilogue, a strided block on the two-pass N_T=128 kernel with a 1x1 strided shortcut, and the
    linear layer as a 1x1 conv (N_T=16)."""
    ini = models._Init(4)
    layers = [ini.conv("stem", 3, 64, 3, 1, 1), nn.Relu(0)]
    layers += models._basic_block(ini, "b1", 64, 64, 1, 1)
    layers += models._basic_block(ini, "b2", 64, 128, 2, 2)
    layers += [nn.AvgPool(4, 4, 4), nn.Flatten(), ini.linear("fc", 128, 10)]
    return nn.ModelSpec(FixedPointConfig(), (3, 8, 8), layers, ini.weights)


@pytest.mark.parametrize("pair", [True, False], ids=["pair", "threads"])
def test_wide_resnet_tma_fused_vs_oracle(pair):
    """Model-level parity through the TMA convs with the fused residual adds (no layer log):
    logits equal the oracle's run_local_forward exactly (batch 3: a partial TMA box)."""
    model = _wide_resnet()
    windows = [(22, 14), (64, 0), (20, 6)]
    x_f = np.random.default_rng(8).uniform(0, 1, (3, 3, 8, 8))
    cfg = nn.ReluConfig([BitWindow(*w) for w in windows])
    layers = [nn._layer_to_json(L) for L in model.layers]
    want, traces, _ = ON.run_local_forward(layers, model.input_shape, model.weights, windows, x_f, 11)
    logits, meters, logs, _ = nn.run_local_forward(model, cfg, x_f, 11, pair=pair, layer_logs=False)
    assert np.array_equal(logits, want)
    assert [tuple(t) for t in meters[0].trace] == [tuple(t) for t in traces[0]]
    assert logs == ([], [])
    # and with the per-layer log (unfused adds) the same logits
    logits2, _, logs2, _ = nn.run_local_forward(model, cfg, x_f, 11, pair=pair)
    assert np.array_equal(logits2, want) and len(logs2[0]) > 0


def test_layer_times_leave_the_forward_unchanged():
    """model_forward_pair(layer_times=...) records one CUDA-event device time per layer (every
    nesting level) and returns the same shares as the untimed forward (fused residual path)."""
    from paper_2309_04875_b200 import ring, sharing, transport
    from paper_2309_04875_b200.protocol import ProtocolSession

    model = _wide_resnet()
    cfg = nn.ReluConfig([BitWindow(22, 14), BitWindow(64, 0), BitWindow(20, 6)])
    x_f = np.random.default_rng(8).uniform(0, 1, (3, 3, 8, 8))
    enc = ring.encode_array(x_f, model.fixed_point)
    s0, s1 = sharing.share_arith(enc, 64, np.random.default_rng(2))
    outs = []
    for times in (None, []):
        stores = nn.build_stores(model, cfg, 3, 5)
        eps = transport.local_pair()
        sess = (ProtocolSession(eps[0], stores[0], model.fixed_point),
                ProtocolSession(eps[1], stores[1], model.fixed_point))
        outs.append(nn.model_forward_pair(sess, s0, s1, model, cfg, layer_times=times))
        if times is not None:
            kinds = [t["kind"] for t in times]
            assert "relu" in kinds and "residual" in kinds and all(t["ms"] >= 0 for t in times)
            top = [t for t in times if "." not in t["layer"]]
            assert len(top) == len(model.layers)
    for a, b in zip(outs[0], outs[1]):
        assert np.array_equal(np.asarray(a.data), np.asarray(b.data))


def test_resnet18_forward_smoke():
    """Full ResNet18-CIFAR at batch 2: runs, spends the analytic rounds, and the logits
    track the plaintext fixed-point forward (fidelity, not exactness: local truncation)."""
    model = models.resnet18_cifar(0)
    cfg = models.resnet_relu_config(model, BitWindow(64, 0))
    x_f = np.random.default_rng(1).uniform(0, 1, (2, 3, 32, 32))
    logits, meters, logs, _ = nn.run_local_forward(model, cfg, x_f, 3)
    assert logits.shape == (2, 10) and np.all(np.isfinite(logits))
    assert meters[0].rounds["Circuit"] == 6 * 17 and meters[0].rounds["Mult"] == 17
    # float reference forward with the same weights (BN folded) and exact ReLU
    ref = _float_forward(model, x_f)
    assert np.max(np.abs(logits - ref)) < 0.05


def _float_forward(model, x):
    import torch.nn.functional as F

    def run(layers, t):
        for L in layers:
            if isinstance(L, nn.Conv2d):
                t = F.conv2d(t, torch.from_numpy(model.weights[L.weight]).double(),
                             torch.from_numpy(model.weights[L.bias]).double(), L.stride, L.pad)
            elif isinstance(L, nn.Relu):
                t = torch.relu(t)
            elif isinstance(L, nn.Residual):
                t = run(L.body, t) + run(L.shortcut, t)
            elif isinstance(L, nn.AvgPool):
                t = F.avg_pool2d(t, (L.kh, L.kw), L.stride)
            elif isinstance(L, nn.Flatten):
                t = t.reshape(t.shape[0], -1)
            elif isinstance(L, nn.Linear):
                t = t @ torch.from_numpy(model.weights[L.weight]).double().T + torch.from_numpy(
                    model.weights[L.bias]).double()
        return t

    return run(model.layers, torch.from_numpy(np.asarray(x, dtype=np.float64))).numpy()


def test_limb_gemm_exact_at_resnet_width():
    """The int8-limb ring GEMM equals uint64 numpy matmul at K = 4608 (ResNet18's largest)."""
    rng = np.random.default_rng(2)
    x = np.frombuffer(rng.bytes(8 * 40 * 4608), dtype="<u8").copy().reshape(40, 4608)
    w = rng.normal(0, 0.05, (24, 4608)).astype(np.float32)
    b = rng.normal(0, 0.1, 24).astype(np.float32)
    for p in (0, 1):
        y = nn.linear_forward(_Sess, ArithShareTensor(p, 64, x), w, b)
        assert np.array_equal(y.data, ON.linear(x, p, w, b))


def _conv_geometries(model):
    """Every distinct conv of a model: (cin, cout, k, stride, pad, H, W, weight name), H x W its input."""
    seen, out = set(), []

    def walk(layers, shape):
        for L in layers:
            if isinstance(L, nn.Residual):
                walk(L.body, shape)
                walk(L.shortcut, shape)
                shape = nn._out_shape(L.body, shape)
                continue
            if isinstance(L, nn.Conv2d):
                key = (L.in_channels, L.out_channels, L.kh, L.stride, L.pad, shape[1], shape[2])
                if key not in seen:
                    seen.add(key)
                    out.append(key + (L.weight, L.bias))
            shape = nn._layer_shape(L, shape)

    walk(model.layers, model.input_shape)
    return out


def _conv_cases():
    cases = []
    for name, model, batch in (("rn18", models.resnet18_cifar(0), 2), ("rn50", models.resnet50(0), 1)):
        for g in _conv_geometries(model):
            cases.append(pytest.param(model, batch, g, id=f"{name}-c{g[0]}-o{g[1]}-k{g[2]}-s{g[3]}-{g[5]}x{g[6]}"))
    return cases


@pytest.mark.parametrize("model,batch,geom", _conv_cases())
def test_every_resnet_conv_bit_exact(model, batch, geom):
    """Every distinct ResNet18-CIFAR and ResNet50 (64x64) conv through nn.conv2d_forward -- the TMA
    tcgen05 kernel (one-pass N_T = 64, two-pass N_T = 128 for N >= 128 at K up to 4608), the stem
    through im2col limb planes, strided 1x1 shortcuts -- equals the reference conv
    (nn.py:227-243, restated in oracle/hb_oracle_nn.conv2d) share for share, both parties."""
    cin, cout, k, stride, pad, h, w, wname, bname = geom
    rng = np.random.default_rng(cin * 1000 + cout + h)
    x = np.frombuffer(rng.bytes(8 * batch * cin * h * w), dtype="<u8").copy().reshape(batch, cin, h, w)
    wt, bias = model.weights[wname], model.weights[bname] + np.float32(0.01)
    layer = nn.Conv2d(cin, cout, k, k, stride, pad, weight="w", bias="b")
    for p in (0, 1):
        y = nn.conv2d_forward(_Sess, ArithShareTensor(p, 64, x), layer, wt, bias)
        want = ON.conv2d(x, p, cin, cout, k, k, stride, pad, wt, bias)
        assert np.array_equal(np.asarray(y.data), want), (geom, p)


def _deep_block_model(cin, cout, side):
    """One ResNet18 down-sampling basic block (3x3 stride-2 conv, 3x3 conv, strided 1x1 shortcut, the
    residual add fused into the second conv's epilogue) at layer3 / layer4 geometry."""
    ini = models._Init(6)
    layers = models._basic_block(ini, "blk", cin, cout, 2, 0)
    layers += [nn.AvgPool(side // 2, side // 2, side // 2), nn.Flatten(), ini.linear("fc", cout, 10)]
    return nn.ModelSpec(FixedPointConfig(), (cin, side, side), layers, ini.weights)


@pytest.mark.parametrize("cin,cout,side", [(128, 256, 16), (256, 512, 8)], ids=["layer3", "layer4"])
def test_fused_residual_block_at_layer3_layer4_geometry(cin, cout, side):
    """The two-pass k_conv_tma<128, 2, J> with the fused residual epilogue at ResNet18 layer3 / layer4
    shapes (K = 1152 / 2304 / 4608): logits equal the oracle's run_local_forward exactly."""
    model = _deep_block_model(cin, cout, side)
    x_f = np.random.default_rng(cin).uniform(0, 1, (2, cin, side, side))
    cfg = nn.ReluConfig([BitWindow(22, 14)])
    layers = [nn._layer_to_json(L) for L in model.layers]
    want, _, _ = ON.run_local_forward(layers, model.input_shape, model.weights, [(22, 14)], x_f, 5)
    logits, _, _, _ = nn.run_local_forward(model, cfg, x_f, 5, pair=True, layer_logs=False)
    assert np.array_equal(logits, want)


@pytest.mark.parametrize("model,batch,geom", _conv_cases())
def test_every_resnet_conv_pair_launch_bit_exact(model, batch, geom):
    """Both parties' convs of a layer in ONE launch (hb_conv_limbs_tma_pair: party 0 and party 1
    tiles on one persistent grid, each with its own tensor maps, truncation, bias and residual)
    equal the reference conv per party -- plus the residual share when one is fused."""
    cin, cout, k, stride, pad, h, w, wname, bname = geom
    if cin % 64:
        pytest.skip("the stem runs through im2col planes, one launch per party")
    rng = np.random.default_rng(cin * 7 + cout + h)
    xs = [np.frombuffer(rng.bytes(8 * batch * cin * h * w), dtype="<u8").copy().reshape(batch, cin, h, w)
          for _ in range(2)]
    wt, bias = model.weights[wname], model.weights[bname] + np.float32(0.01)
    layer = nn.Conv2d(cin, cout, k, k, stride, pad, weight="w", bias="b")
    lw = nn._weight(wt, bias, FixedPointConfig())
    want = [ON.conv2d(x, p, cin, cout, k, k, stride, pad, wt, bias) for p, x in enumerate(xs)]
    ds = [torch.from_numpy(x.view(np.int64)).cuda() for x in xs]
    for fused in (False, True):
        res = None
        if fused:
            res = [torch.from_numpy(rng.integers(0, 2**63, want[0].shape, dtype=np.uint64).view(np.int64)).cuda()
                   for _ in range(2)]
        nn._PLANES.clear()
        out = nn._conv_pair_dev(ds, "nchw", layer, lw, (0, 1), 16, res)
        assert out is not None
        for p in (0, 1):
            got = out[p].cpu().numpy().view(np.uint64)
            exp = want[p] if res is None else want[p] + res[p].cpu().numpy().view(np.uint64)
            assert np.array_equal(got, exp), (geom, p, fused)
    nn._PLANES.clear()


def test_resnet18_full_forward_bit_exact_vs_oracle():
    """The whole ResNet18-CIFAR private inference (batch 1, the benchmark's per-group 8-bit windows,
    fused residual adds, paired conv launches, every ReLU through the fused pair kernel) equals the
    oracle's run_local_forward (the reference algorithm restated, with Residual) exactly -- logits
    and both parties' meter traces."""
    model = models.resnet18_cifar(0)
    wins = [(17, 9), (18, 10), (18, 10), (19, 11), (20, 12)]  # configs/resnet18_windows_w8.json
    cfg = nn.ReluConfig([BitWindow(*w) for w in wins])
    x_f = np.random.default_rng(33).uniform(0, 1, (1, 3, 32, 32))
    layers = [nn._layer_to_json(L) for L in model.layers]
    want, traces, _ = ON.run_local_forward(layers, model.input_shape, model.weights, wins, x_f, 29)
    logits, meters, _, _ = nn.run_local_forward(model, cfg, x_f, 29, pair=True, layer_logs=False)
    assert np.array_equal(logits, want)
    for p in (0, 1):
        assert [tuple(t) for t in meters[p].trace] == [tuple(t) for t in traces[p]]


def test_resnet50_full_forward_bit_exact_vs_oracle():
    """The whole ResNet50 (64x64, CIFAR stem) private inference at batch 1 with the benchmark's
    per-group 8-bit windows equals the oracle's run_local_forward exactly (bottleneck blocks, 1x1
    convs up to 2048 channels, the N_T = 128 two-pass kernel at K up to 4608)."""
    model = models.resnet50(0)
    wins = [(17, 9), (18, 10), (20, 12), (22, 14), (23, 15)]  # configs/resnet50_windows_w8.json
    cfg = nn.ReluConfig([BitWindow(*w) for w in wins])
    x_f = np.random.default_rng(34).uniform(0, 1, (1, 3, 64, 64))
    layers = [nn._layer_to_json(L) for L in model.layers]
    want, traces, _ = ON.run_local_forward(layers, model.input_shape, model.weights, wins, x_f, 31)
    logits, meters, _, _ = nn.run_local_forward(model, cfg, x_f, 31, pair=True, layer_logs=False)
    assert np.array_equal(logits, want)
    assert [tuple(t) for t in meters[0].trace] == [tuple(t) for t in traces[0]]
