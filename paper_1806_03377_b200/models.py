"""Model specs the executor can run, their synthetic data and their layer profiles.

The reference models a network only as a chain of ``LayerProfile`` rows
(profiles.py:24-89) and its numerics only as the linear toy of
semantics.py:39-116.  The B200 executor runs real layers; profile layer l
(1-based) is ``Linear(widths[l-1] -> widths[l])`` followed by ReLU for every
layer but the last, and the loss is the mean-over-batch squared error
L = 1/(2B) * sum_b ||Z_b - T_b||^2 (the paper averages over the minibatch,
PAPER.md:623-624; the toy's 0.5*||r||^2 sum is its B=1 case).

Synthetic data follows semantics.py:76-80 and 93-116: one seeded
``numpy.random.default_rng(seed)`` (PCG64) stream, ``n_blocks`` input/target
blocks, minibatch m uses block (m-1) % n_blocks.  Weights ~ N(0, 2/d_in)
(He), biases ~ N(0, 0.01^2), inputs and targets ~ N(0, 1).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .errors import ValidationError
from .profiles import HardwareSpec, LayerProfile, ModelProfile, build_context

DTYPES = ("fp32", "bf16")


@dataclass(frozen=True)
class MLPSpec:
    widths: tuple[int, ...]  # d_0 .. d_L
    batch: int = 32
    dtype: str = "fp32"
    lr: float = 1e-3
    n_blocks: int = 8
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "widths", tuple(int(w) for w in self.widths))
        if len(self.widths) < 2:
            raise ValidationError("an MLP needs at least one layer (two widths)")
        if any(w < 1 for w in self.widths) or self.batch < 1 or self.n_blocks < 1:
            raise ValidationError("widths, batch and n_blocks must be positive")
        if self.dtype not in DTYPES:
            raise ValidationError(f"dtype must be one of {DTYPES}, got {self.dtype!r}")
        if self.lr < 0:
            raise ValidationError("lr must be >= 0")
        if self.dtype == "bf16" and any(w % 8 for w in self.widths):
            raise ValidationError("bf16 layers need widths that are multiples of 8 (16-byte TMA rows)")

    @property
    def num_layers(self) -> int:
        return len(self.widths) - 1

    @property
    def bytes_per_elem(self) -> int:
        return 4 if self.dtype == "fp32" else 2

    def flops_per_sample(self) -> float:
        """Algorithmic fwd+bwd FLOPs per sample: 6 * sum(d_in*d_out) minus the unneeded first dgrad."""
        macs = [a * b for a, b in zip(self.widths[:-1], self.widths[1:])]
        return 6.0 * sum(macs) - 2.0 * macs[0]


def mlp(width: int, layers: int, **kw) -> MLPSpec:
    return MLPSpec(widths=(width,) * (layers + 1), **kw)


def init_params(spec: MLPSpec) -> list[tuple[np.ndarray, np.ndarray]]:
    """Initial (W [out,in], b [out]) per layer, fp64, from the spec's seeded stream."""
    rng = np.random.default_rng(spec.seed)
    out = []
    for din, dout in zip(spec.widths[:-1], spec.widths[1:]):
        W = rng.normal(0.0, np.sqrt(2.0 / din), size=(dout, din))
        b = rng.normal(0.0, 0.01, size=dout)
        out.append((W, b))
    return out


def make_data(spec: MLPSpec) -> tuple[np.ndarray, np.ndarray]:
    """(X [n_blocks, B, d_0], T [n_blocks, B, d_L]) fp64; drawn after the parameters."""
    rng = np.random.default_rng([spec.seed, 1])
    X = rng.normal(0.0, 1.0, size=(spec.n_blocks, spec.batch, spec.widths[0]))
    T = rng.normal(0.0, 1.0, size=(spec.n_blocks, spec.batch, spec.widths[-1]))
    return X, T


def mlp_profile(spec: MLPSpec, tflops: float = 1000.0) -> ModelProfile:
    """Analytic per-layer profile (times from FLOPs at ``tflops``) for planning / prediction."""
    layers = []
    for l, (din, dout) in enumerate(zip(spec.widths[:-1], spec.widths[1:]), start=1):
        f = 2.0 * spec.batch * din * dout / (tflops * 1e12)
        layers.append(LayerProfile(l, f"linear{l}", f, 2.0 * f, spec.batch * dout, din * dout + dout))
    return ModelProfile(layers=tuple(layers), minibatch_size=spec.batch)


def mlp_context(spec: MLPSpec, machines: int = 1, bandwidth: float = 770e9, tflops: float = 1000.0):
    """CostContext for an MLP spec (bandwidth default: measured B200 NVLink peer copy)."""
    return build_context(mlp_profile(spec, tflops), HardwareSpec(machines, bandwidth, spec.bytes_per_elem))


# ---------------------------------------------------------------- convolutional networks (configs[2])
@dataclass(frozen=True)
class LayerDef:
    """One profile layer of a ConvNetSpec: a 3x3/pad-1 convolution (+ReLU, optional 2x2 max pool)
    or a Linear layer (+ReLU unless it is the model output)."""

    kind: str  # "conv" | "linear"
    c_out: int
    pool: bool = False


@dataclass(frozen=True)
class LayerGeom:
    kind: str
    h: int  # conv input spatial size
    w: int
    c_in: int  # channels (conv) / features (linear)
    c_out: int
    pool: bool
    relu: bool
    im2col: bool  # first conv on an image with < 64 channels
    in_features: int
    out_features: int  # per-sample, after pooling
    pre_features: int  # per-sample, before pooling
    w_shape: tuple[int, int]  # conv: Wt [9*c_in (or 64), c_out]; linear: [c_out, c_in]; transformer: flat
    ffn: int = 0  # transformer block hidden width
    vocab: int = 0  # head: valid vocabulary (c_out is the padded one)

    @property
    def w_numel(self) -> int:
        return self.w_shape[0] * self.w_shape[1]

    @property
    def b_numel(self) -> int:
        if self.kind == "embed":
            return 0
        if self.kind == "block":
            return 9 * self.c_in + self.ffn
        if self.kind == "head":
            return 2 * self.c_in
        return self.c_out

    @property
    def macs_per_sample(self) -> int:
        """Multiply-adds of the forward pass per sample (algorithmic, unpadded)."""
        if self.kind == "conv":
            return self.h * self.w * 9 * self.c_in * self.c_out
        return self.c_in * self.c_out


@dataclass(frozen=True)
class ConvNetSpec:
    """A VGG-style network: NHWC bf16 images, conv/pool feature stack, Linear classifier, softmax
    cross-entropy (mean over the minibatch).  Profile layer l (1-based) is ``layers[l-1]``; pools
    belong to the convolution they follow (PipeDream's VGG-16 has 16 profile layers)."""

    image: tuple[int, int, int]  # (H, W, C)
    layers: tuple[LayerDef, ...]
    batch: int = 32
    dtype: str = "bf16"
    lr: float = 1e-3
    n_blocks: int = 4
    seed: int = 0

    def __post_init__(self):
        object.__setattr__(self, "layers", tuple(self.layers))
        if self.dtype != "bf16":
            raise ValidationError("convolutional networks run in bf16 (tcgen05)")
        if not self.layers or self.layers[-1].kind != "linear":
            raise ValidationError("the model output must be a Linear layer (softmax cross-entropy)")
        self.geoms()  # validates the shapes

    @property
    def num_layers(self) -> int:
        return len(self.layers)

    @property
    def bytes_per_elem(self) -> int:
        return 2

    @property
    def classes(self) -> int:
        return self.layers[-1].c_out

    def geoms(self) -> list[LayerGeom]:
        h, w, c = self.image
        out, flat = [], False
        for i, ld in enumerate(self.layers):
            last = i == len(self.layers) - 1
            if ld.kind == "conv":
                if flat:
                    raise ValidationError("conv after a linear layer")
                im2col = i == 0 and c < 64
                if not im2col and c % 64:
                    raise ValidationError(f"layer {i + 1}: conv input channels must be a multiple of 64 (got {c})")
                if ld.c_out % 64:
                    raise ValidationError(f"layer {i + 1}: conv output channels must be a multiple of 64")
                if im2col and 9 * c > 64:
                    raise ValidationError("the im2col'ed image layer supports at most 7 input channels")
                if ld.pool and (h % 2 or w % 2):
                    raise ValidationError(f"layer {i + 1}: pooling needs even spatial sizes")
                ho, wo = (h // 2, w // 2) if ld.pool else (h, w)
                out.append(LayerGeom("conv", h, w, c, ld.c_out, ld.pool, True, im2col, h * w * c, ho * wo * ld.c_out,
                                     h * w * ld.c_out, ((64 if im2col else 9 * c), ld.c_out)))
                h, w, c = ho, wo, ld.c_out
            elif ld.kind == "linear":
                fin = h * w * c
                if ld.c_out % 8 or fin % 8:
                    raise ValidationError(f"layer {i + 1}: linear widths must be multiples of 8")
                out.append(LayerGeom("linear", 1, 1, fin, ld.c_out, False, not last, False, fin, ld.c_out, ld.c_out,
                                     (ld.c_out, fin)))
                h, w, c, flat = 1, 1, ld.c_out, True
            else:
                raise ValidationError(f"unknown layer kind {ld.kind!r}")
        return out

    @property
    def widths(self) -> tuple[int, ...]:
        """Per-sample features at every layer boundary (d_0 = the image)."""
        g = self.geoms()
        return (g[0].in_features,) + tuple(x.out_features for x in g)

    def n_params(self) -> int:
        return sum(x.w_numel + x.c_out for x in self.geoms())

    def flops_per_sample(self) -> float:
        """Algorithmic fwd+bwd FLOPs per sample (6 x MACs), minus the first layer's unneeded dgrad."""
        macs = [x.macs_per_sample for x in self.geoms()]
        return 6.0 * sum(macs) - 2.0 * macs[0]


def vgg16(batch: int = 32, classes: int = 1000, image: int = 224, **kw) -> ConvNetSpec:
    """VGG-16 (13 conv + 5 max pool + 3 FC), the network of BASELINE configs[2] / PAPER.md:816."""
    cfg = [64, 64, "P", 128, 128, "P", 256, 256, 256, "P", 512, 512, 512, "P", 512, 512, 512, "P"]
    layers = []
    for v in cfg:
        if v == "P":
            layers[-1] = LayerDef("conv", layers[-1].c_out, pool=True)
        else:
            layers.append(LayerDef("conv", v))
    layers += [LayerDef("linear", 4096), LayerDef("linear", 4096), LayerDef("linear", classes)]
    return ConvNetSpec(image=(image, image, 3), layers=tuple(layers), batch=batch, **kw)


# ---------------------------------------------------------------- GPT-2 (configs[3])
@dataclass(frozen=True)
class GPTSpec:
    """GPT-2-style decoder: token + position embedding, pre-LN blocks (causal attention with
    64-wide heads, tanh-GELU MLP), final LayerNorm and an (untied) LM head trained with next-token
    softmax cross-entropy (mean over tokens).  Profile layers: 1 = embedding, 2..L+1 = blocks,
    L+2 = head.  The head is untied from the token embedding because they live on different
    pipeline stages (PipeDream keeps one copy of each parameter per stage).  The vocabulary is
    padded to a multiple of 128 (50257 -> 50304); padded logits are excluded from the softmax."""

    vocab: int = 50257
    d: int = 1024
    heads: int = 16
    layers: int = 24
    seq: int = 1024
    ffn: int = 0  # 0: 4*d
    batch: int = 8  # sequences per minibatch
    dtype: str = "bf16"
    lr: float = 1e-4
    n_blocks: int = 2
    seed: int = 0

    def __post_init__(self):
        if self.ffn == 0:
            object.__setattr__(self, "ffn", 4 * self.d)
        if self.dtype != "bf16":
            raise ValidationError("transformer stages run in bf16 (tcgen05)")
        if self.d != 64 * self.heads:
            raise ValidationError("head dim must be 64 (d == 64 * heads)")
        if self.d % 256 or self.d > 2048:
            raise ValidationError("d must be a multiple of 256 and <= 2048 (LayerNorm kernel)")
        if self.seq % 128:
            raise ValidationError("seq must be a multiple of 128 (attention tiles)")
        if self.ffn % 8:
            raise ValidationError("ffn must be a multiple of 8")

    @property
    def vocab_pad(self) -> int:
        return -(-self.vocab // 128) * 128

    @property
    def num_layers(self) -> int:
        return self.layers + 2

    @property
    def bytes_per_elem(self) -> int:
        return 2

    @property
    def tokens(self) -> int:
        return self.batch * self.seq

    def geoms(self) -> list[LayerGeom]:
        S, d, f, Vp = self.seq, self.d, self.ffn, self.vocab_pad
        emb = LayerGeom("embed", S, self.heads, Vp, d, False, False, False, S, S * d, S * d, (Vp + S, d))
        blk = LayerGeom("block", S, self.heads, d, d, False, False, False, S * d, S * d, S * d, (4 * d + 2 * f, d),
                        ffn=f)
        head = LayerGeom("head", S, self.heads, d, Vp, False, False, False, S * d, S * Vp, S * d, (Vp, d),
                         vocab=self.vocab)
        return [emb] + [blk] * self.layers + [head]

    @property
    def widths(self) -> tuple[int, ...]:
        g = self.geoms()
        return (self.seq,) + tuple(x.out_features for x in g)

    def n_params(self) -> int:
        return sum(x.w_numel + x.b_numel for x in self.geoms())

    def flops_per_sample(self) -> float:
        """Algorithmic fwd+bwd FLOPs per sequence: 6 x (linear MACs + causal attention S^2 d + head)."""
        S, d, f = self.seq, self.d, self.ffn
        block = S * (4 * d * d + 2 * d * f) + S * S * d
        return 6.0 * (self.layers * block + S * d * self.vocab)


def gpt2_medium(batch: int = 8, seq: int = 1024, **kw) -> GPTSpec:
    """GPT-2 medium: 24 layers, d 1024, 16 heads, vocab 50257 (BASELINE configs[3])."""
    return GPTSpec(vocab=50257, d=1024, heads=16, layers=24, seq=seq, batch=batch, **kw)


def init_params_any(spec) -> list[tuple[np.ndarray, np.ndarray]]:
    """Initial parameters of an MLP or ConvNet spec, fp64.  Conv weights are stored tap-major
    Wt [9*c_in, c_out] (row (r*3+s)*c_in + c); the im2col'ed image layer pads rows 9*c_in..63
    with zeros.  He-normal weights, N(0, 0.01^2) biases, one seeded PCG64 stream."""
    if isinstance(spec, MLPSpec):
        return init_params(spec)
    rng = np.random.default_rng(spec.seed)
    out = []
    if isinstance(spec, GPTSpec):
        d, f, Vp, S = spec.d, spec.ffn, spec.vocab_pad, spec.seq
        proj = 0.02 / np.sqrt(2.0 * spec.layers)
        for g in spec.geoms():
            if g.kind == "embed":
                W = np.concatenate([rng.normal(0.0, 0.02, size=(Vp, d)), rng.normal(0.0, 0.01, size=(S, d))])
                out.append((W, np.zeros(0)))
            elif g.kind == "block":
                W = np.concatenate([rng.normal(0.0, 0.02, size=3 * d * d), rng.normal(0.0, proj, size=d * d),
                                    rng.normal(0.0, 0.02, size=f * d), rng.normal(0.0, proj, size=d * f)])
                b = np.concatenate([np.zeros(3 * d + d + f + d), np.ones(d), np.zeros(d), np.ones(d), np.zeros(d)])
                out.append((W.reshape(g.w_shape), b))
            else:
                out.append((rng.normal(0.0, 0.02, size=g.w_shape), np.concatenate([np.ones(d), np.zeros(d)])))
        return out
    for g in spec.geoms():
        if g.kind == "conv":
            fan = 9 * g.c_in
            W = np.zeros(g.w_shape)
            W[:fan] = rng.normal(0.0, np.sqrt(2.0 / fan), size=(fan, g.c_out))
        else:
            W = rng.normal(0.0, np.sqrt(2.0 / g.c_in), size=g.w_shape)
        out.append((W, rng.normal(0.0, 0.01, size=g.c_out)))
    return out


def make_data_any(spec):
    """MLP: (X, T) as make_data.  ConvNet: images X [n_blocks, B, H, W, C] ~ N(0, 1) (fp64) and
    labels [n_blocks, B] uniform over the classes (int32)."""
    if isinstance(spec, MLPSpec):
        return make_data(spec)
    rng = np.random.default_rng([spec.seed, 1])
    if isinstance(spec, GPTSpec):  # next-token prediction on synthetic token streams
        tok = rng.integers(0, spec.vocab, size=(spec.n_blocks, spec.batch, spec.seq + 1)).astype(np.int32)
        return tok[:, :, :-1].copy(), tok[:, :, 1:].copy()
    H, W, C = spec.image
    X = rng.normal(0.0, 1.0, size=(spec.n_blocks, spec.batch, H, W, C))
    y = rng.integers(0, spec.classes, size=(spec.n_blocks, spec.batch)).astype(np.int32)
    return X, y
