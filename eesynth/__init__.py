"""Seeded synthetic inputs shared by the oracle tests and the CUDA path.

This module holds NONE of the method's arithmetic: it only draws seeded random
numbers with the shapes and value distributions of the paper's workloads
(Llama-2 7B/13B/70B exit heads, batch 16 x seq 2048) and rounds
them to bf16 storage.  The recipe is stated in DESIGN.md §4.

Every generator is a pure function of (config, seed, n_tokens): generating on
the CPU gives bit-identical bytes for both sides of a parity test; generating
on the GPU (bench, full-size sampled parity) uses torch's CUDA Philox stream,
which is deterministic for a given seed on a given device.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import torch

# BASELINE.json configs.  `after` = backbone layer each exit
# is attached to (1/4 depth / evenly spaced, A18).
CONFIGS = {
    "tiny": dict(hidden=64, vocab=512, ffn=0, arch="norm", tokens=256, layers=2,
                 after=[1, 2], init="copy", seed=0),
    "7b": dict(hidden=4096, vocab=32000, ffn=0, arch="embedding", tokens=8 * 2048,
               layers=32, after=[8, 16], init="copy", seed=1),
    "13b": dict(hidden=5120, vocab=32000, ffn=13824, arch="mlp", tokens=16 * 2048,
                layers=40, after=[10, 20, 30, 40], init="copy", seed=2),
    "70b": dict(hidden=8192, vocab=32000, ffn=28672, arch="mlp", tokens=32 * 2048,
                layers=80, after=[20, 40, 60, 80], init="copy", seed=3),
    "70b_dp": dict(hidden=8192, vocab=32000, ffn=28672, arch="mlp", tokens=32 * 2048,
                   layers=80, after=[10, 20, 30, 40, 50, 60, 70, 80], init="copy", seed=4),
    # Layer exits (NEXT #2): a full Llama-2 layer per exit; tokens are
    # whole sequences (causal attention within each).
    "tiny_layer": dict(hidden=256, vocab=1000, ffn=384, arch="layer", tokens=2 * 128, layers=2,
                       after=[1, 2], init="copy", seed=5, n_heads=2, n_kv_heads=1, seq_len=128),
    # the paper's end-to-end 13B conversion: ONE MLP exit
    # at 1/4 depth, batch 16 x 2048 -- the --parallel pp bench runs the frozen
    # backbone's partial forward (layers 1..10) and the exit's tuning
    "13b_q": dict(hidden=5120, vocab=32000, ffn=13824, arch="mlp", tokens=16 * 2048,
                  layers=40, after=[10], init="random", seed=7),
    "70b_q": dict(hidden=8192, vocab=32000, ffn=28672, arch="mlp", tokens=16 * 2048,
                  layers=80, after=[20], init="random", seed=8),
    # the paper's architecture comparison: 13B with 8 exits at 1/8 .. 8/8 depth
    # (P:465), batch 16 x 2048
    "13b_layer": dict(hidden=5120, vocab=32000, ffn=13824, arch="layer", tokens=16 * 2048,
                      layers=40, after=[5, 10, 15, 20, 25, 30, 35, 40], init="copy", seed=6,
                      n_heads=40, n_kv_heads=40, seq_len=2048),
}

MATRIX_STD = 0.02          # N(0, 0.02^2) weights (A12)
GAIN_JITTER = 0.1          # norm gains 1 + 0.1 N(0,1)
MASSIVE_CHANNELS = 4       # Llama residual-stream outlier channels
MASSIVE_SCALE = 50.0


@dataclass
class Cfg:
    name: str
    hidden: int
    vocab: int
    ffn: int
    arch: str
    tokens: int
    layers: int
    after: list
    init: str
    seed: int
    n_heads: int = 0          # Layer exits: attention geometry (head dim 128)
    n_kv_heads: int = 0
    seq_len: int = 0
    exits: int = field(init=False)

    def __post_init__(self):
        self.exits = len(self.after)


def get_cfg(name: str, **over) -> Cfg:
    d = dict(CONFIGS[name])
    d.update(over)
    if "after" in over or "exits" in over:
        pass
    return Cfg(name=name, **d)


def _gen(seed: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed(int(seed))
    return g


def _randn(shape, g, device, std=1.0, mean=0.0):
    t = torch.randn(*shape, generator=g, device=device, dtype=torch.float32)
    if std != 1.0:
        t.mul_(std)
    if mean != 0.0:
        t.add_(mean)
    return t


def hidden_states(cfg: Cfg, n_tokens: int | None = None, seed: int | None = None,
                  device="cpu", dtype=torch.bfloat16):
    """Cached hidden states h_i [N x h] at each exit layer.

    H_l = s_l * N(0, 1), s_l growing with depth (1 at the first exit, 2 at the
    last), plus MASSIVE_CHANNELS fixed channels at MASSIVE_SCALE x RMS for the
    Llama-shaped configs (not for tiny).
    """
    n = cfg.tokens if n_tokens is None else int(n_tokens)
    s = cfg.seed if seed is None else seed
    out = []
    E = cfg.exits
    for i in range(E):
        g = _gen(s * 1000 + 17 * i + 1, device)
        scale = 1.0 + (i / max(E - 1, 1))
        x = _randn((n, cfg.hidden), g, device, std=scale)
        if cfg.name != "tiny" and cfg.hidden >= 256:
            ch = torch.arange(MASSIVE_CHANNELS, device=device) * (cfg.hidden // MASSIVE_CHANNELS) + 7
            x[:, ch] *= MASSIVE_SCALE
        out.append(x.to(dtype))
    return out


def targets(cfg: Cfg, n_tokens: int | None = None, seed: int | None = None, device="cpu",
            ignore_frac: float = 1.0 / 64):
    """Next-token targets [N] int32, uniform over [0, V); a fraction set to -1
    (ignore_index, e.g. padding; A6)."""
    n = cfg.tokens if n_tokens is None else int(n_tokens)
    s = cfg.seed if seed is None else seed
    g = _gen(s * 1000 + 999, device)
    y = torch.randint(0, cfg.vocab, (n,), generator=g, device=device, dtype=torch.int64)
    if ignore_frac > 0:
        drop = torch.rand(n, generator=g, device=device) < ignore_frac
        y = torch.where(drop, torch.full_like(y, -1), y)
    return y.to(torch.int32)


def head_params(cfg: Cfg, seed: int | None = None, device="cpu", w_out_std: float | None = None):
    """Exit-head parameters drawn directly (for parity tests that do not go
    through the initialiser): matrices N(0, 0.02^2) (tiny: W_out N(0, 1/h) for
    O(1) logits), gains 1 + 0.1 N(0,1).  fp32 masters on the bf16 grid, so the
    bf16 operand copy is exact.  Returns a list (one dict per exit)."""
    s = cfg.seed if seed is None else seed
    h, V, F = cfg.hidden, cfg.vocab, cfg.ffn
    if w_out_std is None:
        w_out_std = (1.0 / h) ** 0.5 if cfg.name == "tiny" else MATRIX_STD
    tiny = cfg.name.startswith("tiny")
    mstd = (1.0 / h) ** 0.5 if tiny else MATRIX_STD
    res = []
    for i in range(cfg.exits):
        g = _gen(s * 1000 + 500 + i, device)
        p = {"w_out": _randn((V, h), g, device, std=w_out_std)}
        if cfg.arch != "embedding":
            p["g_f"] = _randn((h,), g, device, std=GAIN_JITTER, mean=1.0)
        if cfg.arch in ("mlp", "layer"):
            p["g_a"] = _randn((h,), g, device, std=GAIN_JITTER, mean=1.0)
            p["w_gate"] = _randn((F, h), g, device, std=mstd)
            p["w_up"] = _randn((F, h), g, device, std=mstd)
            p["w_down"] = _randn((h, F), g, device, std=mstd)
        if cfg.arch == "layer":
            p.update(_attn_params(cfg, g, device))
        for k in list(p):
            p[k] = p[k].to(torch.bfloat16).to(torch.float32)   # on the bf16 grid
        res.append(p)
    return res


def _attn_params(cfg: Cfg, g, device):
    """Attention tensors of a Layer exit / backbone layer.  tiny: W_q, W_k with
    std 2/sqrt(h) (attention scores of std ~4: peaked, so the softmax backward
    is exercised), W_v, W_o 1/sqrt(h); Llama-shaped: N(0, 0.02^2) (score std
    ~2 at h = 5120)."""
    h = cfg.hidden
    hkv = 128 * (cfg.n_kv_heads or cfg.n_heads)
    tiny = cfg.name.startswith("tiny")
    sqk = 2.0 * (1.0 / h) ** 0.5 if tiny else MATRIX_STD
    svo = (1.0 / h) ** 0.5 if tiny else MATRIX_STD
    return {"g_att": _randn((h,), g, device, std=GAIN_JITTER, mean=1.0),
            "w_q": _randn((h, h), g, device, std=sqk), "w_k": _randn((hkv, h), g, device, std=sqk),
            "w_v": _randn((hkv, h), g, device, std=svo), "w_o": _randn((h, h), g, device, std=svo)}


def attn_geometry(cfg: Cfg) -> dict | None:
    """The oracle's `attn` argument for Layer exits (None otherwise)."""
    if cfg.arch != "layer":
        return None
    return {"seq_len": cfg.seq_len, "n_heads": cfg.n_heads,
            "n_kv": cfg.n_kv_heads or cfg.n_heads, "theta": 10000.0}


def backbone(cfg: Cfg, seed: int | None = None, device="cpu"):
    """Synthetic frozen backbone views needed by Copy init (D8): the final norm
    gain, the final output embedding and, for each exit layer, that layer's MLP
    and pre-MLP norm gain (Layer exits: the last layer, attention included).
    bf16 tensors (a Llama checkpoint is bf16)."""
    s = cfg.seed if seed is None else seed
    h, V, F = cfg.hidden, cfg.vocab, cfg.ffn
    g = _gen(s * 1000 + 300, device)
    w_std = (1.0 / h) ** 0.5 if cfg.name == "tiny" else MATRIX_STD
    bb = {
        "final_norm": _randn((h,), g, device, std=GAIN_JITTER, mean=1.0).to(torch.bfloat16),
        "w_out": _randn((V, h), g, device, std=w_std).to(torch.bfloat16),
        "layers": {},
    }
    if cfg.arch == "mlp":
        for k in cfg.after:
            gl = _gen(s * 1000 + 400 + k, device)
            bb["layers"][k] = {
                "mlp_norm": _randn((h,), gl, device, std=GAIN_JITTER, mean=1.0).to(torch.bfloat16),
                "w_gate": _randn((F, h), gl, device, std=MATRIX_STD).to(torch.bfloat16),
                "w_up": _randn((F, h), gl, device, std=MATRIX_STD).to(torch.bfloat16),
                "w_down": _randn((h, F), gl, device, std=MATRIX_STD).to(torch.bfloat16),
            }
    if cfg.arch == "layer":
        gl = _gen(s * 1000 + 400 + cfg.layers, device)
        mstd = (1.0 / h) ** 0.5 if cfg.name.startswith("tiny") else MATRIX_STD
        L = {"mlp_norm": _randn((h,), gl, device, std=GAIN_JITTER, mean=1.0),
             "w_gate": _randn((F, h), gl, device, std=mstd),
             "w_up": _randn((F, h), gl, device, std=mstd),
             "w_down": _randn((h, F), gl, device, std=mstd)}
        L.update(_attn_params(cfg, gl, device))
        bb["layers"][cfg.layers] = {k: v.to(torch.bfloat16) for k, v in L.items()}
    return bb


def to_f64(t: torch.Tensor):
    """Exact widening of a (bf16/fp32) tensor to a float64 numpy array."""
    return t.detach().to("cpu").to(torch.float64).numpy()
