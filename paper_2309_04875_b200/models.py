"""Model builders for private inference.

* ``desk_cnn`` / ``desk_mlp``: the reference's desk models (models.py:33-72),
  same layers and the same seeded random init, so model-level parity can be
  checked against ``ringmpc.cli.run_local_forward`` (the reference trains them
  with numpy SGD; training is out of scope here, the init is what is shared).
* ``resnet18_cifar`` / ``resnet50``: the ResNets of BASELINE.json configs[2-4]
  with random init (torchvision's scheme: Kaiming-normal fan_out convs, default
  Linear init) and BatchNorm folded into the conv (identity statistics at init).
  The reference cannot express these (no residual layer); they
  use ``nn.Residual``.
"""

from __future__ import annotations

import numpy as np

from .nn import AvgPool, Conv2d, Flatten, Linear, ModelSpec, Relu, ReluConfig, Residual
from .ring import BitWindow, FixedPointConfig

N_CLASSES = 10
IMG_SIDE = 8


def desk_mlp(seed: int, fxp: FixedPointConfig | None = None) -> ModelSpec:
    """64-32-10 MLP with the reference's seeded init (models.py:33-47)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x31]))
    d_in, d_h = IMG_SIDE * IMG_SIDE, 32
    w = {
        "fc1.w": rng.normal(0, np.sqrt(2.0 / d_in), (d_h, d_in)).astype(np.float32),
        "fc1.b": np.zeros(d_h, dtype=np.float32),
        "fc2.w": rng.normal(0, np.sqrt(2.0 / d_h), (N_CLASSES, d_h)).astype(np.float32),
        "fc2.b": np.zeros(N_CLASSES, dtype=np.float32),
    }
    layers = [Linear(d_in, d_h, "fc1.w", "fc1.b"), Relu(0), Linear(d_h, N_CLASSES, "fc2.w", "fc2.b")]
    return ModelSpec(fxp or FixedPointConfig(), (d_in,), layers, w)


def desk_cnn(seed: int, fxp: FixedPointConfig | None = None) -> ModelSpec:
    """conv3x3x8 -> pool -> conv3x3x16 -> pool -> linear, reference init (models.py:50-72)."""
    rng = np.random.default_rng(np.random.SeedSequence([seed, 0x32]))
    c1, c2 = 8, 16
    d_fc = c2 * 2 * 2
    w = {
        "conv1.w": rng.normal(0, np.sqrt(2.0 / 9), (c1, 1, 3, 3)).astype(np.float32),
        "conv1.b": np.zeros(c1, dtype=np.float32),
        "conv2.w": rng.normal(0, np.sqrt(2.0 / (9 * c1)), (c2, c1, 3, 3)).astype(np.float32),
        "conv2.b": np.zeros(c2, dtype=np.float32),
        "fc.w": rng.normal(0, np.sqrt(2.0 / d_fc), (N_CLASSES, d_fc)).astype(np.float32),
        "fc.b": np.zeros(N_CLASSES, dtype=np.float32),
    }
    layers = [
        Conv2d(1, c1, 3, 3, 1, 1, "conv1.w", "conv1.b"), Relu(0), AvgPool(2, 2, 2),
        Conv2d(c1, c2, 3, 3, 1, 1, "conv2.w", "conv2.b"), Relu(1), AvgPool(2, 2, 2),
        Flatten(), Linear(d_fc, N_CLASSES, "fc.w", "fc.b"),
    ]
    return ModelSpec(fxp or FixedPointConfig(), (1, IMG_SIDE, IMG_SIDE), layers, w)


# ------------------------------------------------------------------ ResNets
class _Init:
    """torchvision ResNet init with BatchNorm folded (gamma=1, beta=0, mean=0, var=1, eps=1e-5)."""

    BN_SCALE = 1.0 / np.sqrt(1.0 + 1e-5)

    def __init__(self, seed: int):
        self.rng = np.random.default_rng(np.random.SeedSequence([seed, 0x7E5]))
        self.weights: dict = {}

    def conv(self, name: str, cin: int, cout: int, k: int, stride: int, pad: int) -> Conv2d:
        std = np.sqrt(2.0 / (cout * k * k))  # kaiming_normal_(mode="fan_out", nonlinearity="relu")
        self.weights[name + ".w"] = (self.rng.normal(0, std, (cout, cin, k, k)) * self.BN_SCALE).astype(np.float32)
        self.weights[name + ".b"] = np.zeros(cout, dtype=np.float32)  # folded BN bias: beta - mean*scale = 0
        return Conv2d(cin, cout, k, k, stride, pad, name + ".w", name + ".b")

    def linear(self, name: str, fin: int, fout: int) -> Linear:
        bound = 1.0 / np.sqrt(fin)  # nn.Linear default init
        self.weights[name + ".w"] = self.rng.uniform(-bound, bound, (fout, fin)).astype(np.float32)
        self.weights[name + ".b"] = self.rng.uniform(-bound, bound, fout).astype(np.float32)
        return Linear(fin, fout, name + ".w", name + ".b")


def _basic_block(ini, name, cin, cout, stride, group):
    body = (ini.conv(name + ".conv1", cin, cout, 3, stride, 1), Relu(group), ini.conv(name + ".conv2", cout, cout, 3, 1, 1))
    short = () if stride == 1 and cin == cout else (ini.conv(name + ".down", cin, cout, 1, stride, 0),)
    return [Residual(body, short), Relu(group)]


def _bottleneck(ini, name, cin, width, stride, group):
    cout = 4 * width
    body = (ini.conv(name + ".conv1", cin, width, 1, 1, 0), Relu(group),
            ini.conv(name + ".conv2", width, width, 3, stride, 1), Relu(group),
            ini.conv(name + ".conv3", width, cout, 1, 1, 0))
    short = () if stride == 1 and cin == cout else (ini.conv(name + ".down", cin, cout, 1, stride, 0),)
    return [Residual(body, short), Relu(group)]


def resnet18_cifar(seed: int = 0, num_classes: int = 10, side: int = 32, fxp: FixedPointConfig | None = None):
    """CIFAR ResNet18: 3x3 stem (stride 1, no maxpool), 4 stages x 2 basic blocks, global avgpool.

    ReLU groups = the 5 ResNet groups of PAPER.md:451 (stem, layer1..layer4);
    17 ReLUs, 557,056 ReLU elements per 3x32x32 sample."""
    ini = _Init(seed)
    layers = [ini.conv("stem", 3, 64, 3, 1, 1), Relu(0)]
    cin = 64
    for s, (cout, stride) in enumerate(((64, 1), (128, 2), (256, 2), (512, 2))):
        for b in range(2):
            layers += _basic_block(ini, f"layer{s + 1}.{b}", cin, cout, stride if b == 0 else 1, s + 1)
            cin = cout
    final = side // 8
    layers += [AvgPool(final, final, final), Flatten(), ini.linear("fc", 512, num_classes)]
    return ModelSpec(fxp or FixedPointConfig(), (3, side, side), layers, ini.weights)


def resnet50(seed: int = 0, num_classes: int = 200, side: int = 64, fxp: FixedPointConfig | None = None):
    """ResNet50 with the CIFAR-style stem (3x3, stride 1, no maxpool) on side x side inputs
    (BASELINE configs[3]: 3x64x64 TinyImageNet shape; 49 ReLUs)."""
    ini = _Init(seed)
    layers = [ini.conv("stem", 3, 64, 3, 1, 1), Relu(0)]
    cin = 64
    for s, (width, blocks, stride) in enumerate(((64, 3, 1), (128, 4, 2), (256, 6, 2), (512, 3, 2))):
        for b in range(blocks):
            layers += _bottleneck(ini, f"layer{s + 1}.{b}", cin, width, stride if b == 0 else 1, s + 1)
            cin = 4 * width
    final = side // 8
    layers += [AvgPool(final, final, final), Flatten(), ini.linear("fc", 2048, num_classes)]
    return ModelSpec(fxp or FixedPointConfig(), (3, side, side), layers, ini.weights)


def resnet_relu_config(model: ModelSpec, window: BitWindow | None = BitWindow(22, 14)) -> ReluConfig:
    """One window for every ReLU group (the 8-bit reduced ring (22,14) by default: |x| < 2^5 at f=16
    keeps the sign exact (Theorem 1), magnitudes below 2^-2 may be pruned (Theorem 2))."""
    return ReluConfig([window] * model.n_groups)


def conv_macs(model: ModelSpec) -> int:
    """Multiply-accumulates per sample of the model's conv and linear layers (residual branches
    included): the dense contraction the int8-limb ring GEMMs compute (x 15 limb products)."""
    from .nn import _layer_shape

    total = 0

    def visit(layers, cur):
        nonlocal total
        for L in layers:
            nxt = _layer_shape(L, cur)
            if isinstance(L, Conv2d):
                total += nxt[0] * nxt[1] * nxt[2] * L.in_channels * L.kh * L.kw
            elif isinstance(L, Linear):
                total += L.in_features * L.out_features
            elif isinstance(L, Residual):
                visit(L.body, cur)
                visit(L.shortcut, cur)
            cur = nxt

    visit(model.layers, tuple(model.input_shape))
    return total
