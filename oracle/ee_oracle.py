"""EE-Tuning exit-head oracle: plain, slow, fp64 CPU reference.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module.  The product path (``paper_2402_00518_b200``) never imports it, and this
module imports nothing from the product path: the two share no code.

What it computes (citations are PAPER.md line numbers, "P:<line>", plus the
section they fall in; "A<n>" are the readings listed in DESIGN.md §3):

* exit architectures (§2.1 "Architectures of early exits"):
  ``embedding``: logits = z W_out^T with z = x;
  ``norm``:      z = RMSNorm_f(x) (RMSNorm used in experiments P:464);
  ``mlp``:       y = x + MLP(RMSNorm_a(x)), z = RMSNorm_f(y) (pre-norm
                 residual structure P:165-166; SwiGLU MLP as in Llama-2, A2).
  ``layer``:     "a complete Transformer layer, with the same structure as those
                 on the backbone, ... in front of the Norm architecture":
                 x1 = x + W_o attn(RoPE(W_q u1), RoPE(W_k u1), W_v u1),
                 u1 = RMSNorm_att(x); then the MLP exit on x1 (Llama-2 layer,
                 P:356-358; causal attention within each sequence of T tokens).
* loss: next-token negative log-likelihood (§2 "Preliminaries"),
  averaged over valid tokens (A4), ignore_index -1 (A6).
* exits are independent; the backbone is frozen, so gradients flow into the
  exit parameters only and there is no gradient w.r.t. x (P:250-252, P:261,
  §2.2 "Stage 2").
* weighted sum of exit losses: grads of exit i scale by alpha_i (A5).
* Adam with beta1 0.9, beta2 0.95, eps 1e-5 (§3 "Tuning"); SGD.
* LR schedule: linear warmup then linear decay (A14).
* Copy initialisation (§2.1 "Initialization of early exits").

Every floating-point step is fp64 with no tiling, no online softmax and no
recompute: logits are materialised.  ``np.matmul`` is the only library
primitive used for the contractions.  bf16 inputs are widened exactly.

Parity pins for every function live in ``tests/test_oracle_pins.py``.  Random
initialisation is *not* reproduced here (it is pinned statistically on the GPU,
P15 in DESIGN.md) -- "parity unpinned" does not apply to any function below.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

ARCHS = ("embedding", "norm", "mlp", "layer")
MLP_BODY = ("mlp", "layer")
IGNORE_INDEX = -1


# ----------------------------------------------------------------------------
# building blocks
# ----------------------------------------------------------------------------

def bf16_bits_to_f64(bits: np.ndarray) -> np.ndarray:
    """Exact widening of bf16 bit patterns (uint16) to fp64."""
    b = np.ascontiguousarray(bits, dtype=np.uint16).astype(np.uint32) << 16
    return b.view(np.float32).astype(np.float64)


def rmsnorm(x: np.ndarray, g: np.ndarray, eps: float):
    """RMSNorm: out = g * x * r, r = (mean_j x_j^2 + eps)^-1/2.

    Returns (out, r, xhat) with xhat = x * r.
    """
    r = 1.0 / np.sqrt(np.mean(x * x, axis=-1) + eps)
    xhat = x * r[:, None]
    return g[None, :] * xhat, r, xhat


def rmsnorm_backward(dout: np.ndarray, xhat: np.ndarray, r: np.ndarray, g: np.ndarray):
    """Backward of ``rmsnorm`` w.r.t. its input and gain.

    dg = sum_t dout_t * xhat_t;
    dx_t = r_t * (g*dout_t - xhat_t * mean_j(g_j dout_tj xhat_tj)).
    """
    dg = np.sum(dout * xhat, axis=0)
    gd = g[None, :] * dout
    mean_term = np.mean(gd * xhat, axis=-1)
    dx = r[:, None] * (gd - xhat * mean_term[:, None])
    return dx, dg


def sigmoid(a: np.ndarray) -> np.ndarray:
    return 1.0 / (1.0 + np.exp(-a))


def silu(a: np.ndarray) -> np.ndarray:
    """silu(a) = a / (1 + e^-a) (Llama-2 SwiGLU gate, A2)."""
    return a * sigmoid(a)


def silu_grad(a: np.ndarray) -> np.ndarray:
    """d silu / da = sigma(a) * (1 + a (1 - sigma(a)))."""
    s = sigmoid(a)
    return s * (1.0 + a * (1.0 - s))


# ----------------------------------------------------------------------------
# exit head forward
# ----------------------------------------------------------------------------

def _need(params: dict, names, arch):
    for n in names:
        if params.get(n) is None:
            raise ValueError(f"arch {arch!r} requires parameter {n!r}")


def exit_forward(arch: str, params: dict, x: np.ndarray, eps: float, attn: dict | None = None) -> dict:
    """Forward of one exit head up to the logits S = z W_out^T.

    params (fp64 numpy): w_out [V,h]; norm/mlp/layer: g_f [h];
    mlp/layer: g_a [h], w_gate [F,h], w_up [F,h], w_down [h,F];
    layer: g_att [h], w_q [Hq d, h], w_k, w_v [Hkv d, h], w_o [h, Hq d].
    attn (layer only): seq_len T, n_heads Hq, n_kv Hkv, theta (RoPE base).
    """
    if arch not in ARCHS:
        raise ValueError(f"unknown arch {arch!r}")
    _need(params, ["w_out"], arch)
    act = {"x": x}
    xin = x
    if arch == "layer":
        _need(params, ["g_att", "w_q", "w_k", "w_v", "w_o"], arch)
        if attn is None:
            raise ValueError("arch 'layer' needs attn = {seq_len, n_heads, n_kv, theta}")
        xin = _attention_block_forward(params, x, eps, attn, act)
    y = xin
    if arch in MLP_BODY:
        _need(params, ["g_a", "w_gate", "w_up", "w_down"], arch)
        u, r_x, xhat = rmsnorm(xin, params["g_a"], eps)     # pre-norm
        A = u @ params["w_gate"].T
        B = u @ params["w_up"].T
        M = silu(A) * B                                     # SwiGLU (A2)
        y = xin + M @ params["w_down"].T                    # residual
        act.update(u=u, r_x=r_x, xhat=xhat, A=A, B=B, M=M)
    act["y"] = y
    if arch != "embedding":
        _need(params, ["g_f"], arch)
        z, r_y, yhat = rmsnorm(y, params["g_f"], eps)       # Norm exit
        act.update(r_y=r_y, yhat=yhat)
    else:
        z = y                                               # Embedding exit
    act["z"] = z
    act["S"] = z @ params["w_out"].T                        # output embedding
    return act


def _attention_block_forward(params: dict, x: np.ndarray, eps: float, attn: dict,
                             act: dict) -> np.ndarray:
    """Attention half of the Layer exit (Llama-2 layer P:356-358):
    x1 = x + W_o softmax(q k^T / sqrt(d) + causal) v with q, k rotated by RoPE at
    the token's position within its sequence (row % T).  Keeps q, k (rotated),
    v, the attention probabilities P and o for the backward."""
    T, Hq, Hkv = int(attn["seq_len"]), int(attn["n_heads"]), int(attn["n_kv"])
    theta = float(attn.get("theta", 10000.0))
    N, h = x.shape
    if N % T:
        raise ValueError("Layer exit: tokens must be whole sequences of seq_len")
    d = params["w_q"].shape[0] // Hq
    pos = np.arange(N) % T
    u1, r1, xh1 = rmsnorm(x, params["g_att"], eps)
    q = rope((u1 @ params["w_q"].T).reshape(N, Hq, d), pos, theta)
    k = rope((u1 @ params["w_k"].T).reshape(N, Hkv, d), pos, theta)
    v = (u1 @ params["w_v"].T).reshape(N, Hkv, d)
    P = attention_probs(q, k, T)                                    # [B, Hq, T, T]
    g = Hq // Hkv
    o = np.zeros((N, Hq, d))
    for b in range(N // T):
        rs = slice(b * T, (b + 1) * T)
        for j in range(Hq):
            o[rs, j, :] = P[b, j] @ v[rs, j // g, :]
    o = o.reshape(N, Hq * d)
    x1 = x + o @ params["w_o"].T                                    # residual
    act.update(u1=u1, r1=r1, xh1=xh1, q=q, k=k, v=v, P=P, o=o, x1=x1, pos=pos, theta=theta,
               T=T)
    return x1


def attention_probs(q: np.ndarray, k: np.ndarray, T: int) -> np.ndarray:
    """P[b, j] = softmax over keys s <= t of q_t . k_s / sqrt(d) (causal), per
    sequence b and query head j (GQA: kv head j // (Hq / Hkv))."""
    N, Hq, d = q.shape
    g = Hq // k.shape[1]
    P = np.zeros((N // T, Hq, T, T))
    mask = np.triu(np.ones((T, T), dtype=bool), 1)
    for b in range(N // T):
        rs = slice(b * T, (b + 1) * T)
        for j in range(Hq):
            S = q[rs, j, :] @ k[rs, j // g, :].T / math.sqrt(d)
            S = np.where(mask, -np.inf, S)
            E = np.exp(S - S.max(axis=1, keepdims=True))
            P[b, j] = E / E.sum(axis=1, keepdims=True)
    return P


def attention_backward(q, k, v, P, do, T):
    """Backward of o = P v with P = softmax(q k^T / sqrt(d) + causal):
    dv = P^T do;  dP = do v^T;  dS = P * (dP - rowsum(dP * P));
    dq = dS k / sqrt(d);  dk = dS^T q / sqrt(d)  (summed over a GQA group)."""
    N, Hq, d = q.shape
    g = Hq // k.shape[1]
    dq, dk, dv = np.zeros_like(q), np.zeros_like(k), np.zeros_like(v)
    c = 1.0 / math.sqrt(d)
    for b in range(N // T):
        rs = slice(b * T, (b + 1) * T)
        for j in range(Hq):
            Pj = P[b, j]
            dv[rs, j // g, :] += Pj.T @ do[rs, j, :]
            dP = do[rs, j, :] @ v[rs, j // g, :].T
            dS = Pj * (dP - np.sum(dP * Pj, axis=1, keepdims=True))
            dq[rs, j, :] = c * (dS @ k[rs, j // g, :])
            dk[rs, j // g, :] += c * (dS.T @ q[rs, j, :])
    return dq, dk, dv


# ----------------------------------------------------------------------------
# loss
# ----------------------------------------------------------------------------

def lm_loss_stats(S: np.ndarray, targets: np.ndarray) -> dict:
    """Per-token softmax cross-entropy statistics from materialised logits.

    m_t = max_v S_tv; lse_t = m_t + ln sum_v exp(S_tv - m_t);
    loss_t = lse_t - S_{t,y_t} (0 where y_t = -1); conf_t = exp(m_t - lse_t)
    (the maximum softmax probability); argmax_t = lowest v with S_tv = m_t (A9).
    """
    V = S.shape[1]
    t = np.asarray(targets, dtype=np.int64)
    if np.any((t < IGNORE_INDEX) | (t >= V)):
        raise ValueError("target id out of range [-1, V)")
    m = S.max(axis=1)
    lse = m + np.log(np.sum(np.exp(S - m[:, None]), axis=1))
    valid = t != IGNORE_INDEX
    tl = np.where(valid, S[np.arange(S.shape[0]), np.where(valid, t, 0)], 0.0)
    loss = np.where(valid, lse - tl, 0.0)
    conf = np.exp(m - lse)
    argmax = np.argmax(S, axis=1)  # numpy returns the first (lowest) index on ties
    return dict(m=m, lse=lse, loss=loss, conf=conf, argmax=argmax.astype(np.int64),
                valid=valid)


# ----------------------------------------------------------------------------
# one exit: loss and gradients (backprop into exit parameters only)
# ----------------------------------------------------------------------------

@dataclass
class ExitResult:
    loss: float                 # L_i = sum_t w_t loss_t / W  (A4; W global, A16)
    grads: dict                 # same keys as the exit's parameters
    stats: dict                 # per-token lse, loss, conf, argmax
    act: dict = field(repr=False, default_factory=dict)


def exit_loss_and_grads(arch: str, params: dict, x: np.ndarray, targets: np.ndarray,
                        alpha: float, eps: float, valid_count: int | None = None,
                        keep_act: bool = False, weighting="uniform",
                        attn: dict | None = None) -> ExitResult:
    """Loss and parameter gradients of one exit.

    ``valid_count`` is W, the normaliser of the mean over valid tokens; it
    defaults to the number of valid tokens in ``targets`` (single-GPU
    semantics) and is the *global* count under data parallelism (A16).
    The gradient is that of alpha * L_i (A5).

    ``weighting``: "uniform" (w_t = 1 on valid tokens); "confidence" -- the
    dynamic token-wise weights of P:326-336 / App. B.3: w_t = c_t,
    the exit's maximum softmax probability at token t, "detached from the
    computational graph and thus regarded as constants"; or an explicit array
    of per-token constants.  Non-uniform weights are normalised by their sum
    over valid tokens (A17); ``valid_count`` then does not apply.
    """
    act = exit_forward(arch, params, x, eps, attn)
    st = lm_loss_stats(act["S"], targets)
    w = st["valid"].astype(np.float64)
    if isinstance(weighting, str) and weighting == "uniform":
        W = float(np.sum(w)) if valid_count is None else float(valid_count)
    else:
        c = st["conf"] if isinstance(weighting, str) and weighting == "confidence" \
            else np.asarray(weighting, dtype=np.float64)
        if isinstance(weighting, str) and weighting != "confidence":
            raise ValueError(f"unknown weighting {weighting!r}")
        w = w * c                                           # detached constants
        W = float(np.sum(w))
    z = act["z"]
    grads = {k: np.zeros_like(v) for k, v in params.items() if v is not None}
    if W == 0.0:
        return ExitResult(0.0, grads, st, act if keep_act else {})
    loss = float(np.sum(w * st["loss"]) / W)

    # dS_tv = alpha * w_t / W * (softmax(S_t)_v - 1[v = y_t])
    P = np.exp(act["S"] - st["lse"][:, None])
    onehot = np.zeros_like(P)
    rows = np.nonzero(st["valid"])[0]
    onehot[rows, np.asarray(targets)[rows]] = 1.0
    dS = (alpha * w / W)[:, None] * (P - onehot)

    grads["w_out"] = dS.T @ z                               # dW_out = dS^T z
    if arch != "embedding":
        dz = dS @ params["w_out"]                           # dz = dS W_out
        grads.update(exit_body_backward(arch, params, act, dz))
    return ExitResult(loss, grads, st, act if keep_act else {})


def exit_body_backward(arch: str, params: dict, act: dict, dz: np.ndarray) -> dict:
    """Gradients of the exit body below W_out given dz = dL/dz: the
    final RMSNorm gain and, for MLP exits, the SwiGLU MLP and its pre-norm gain;
    for Layer exits also the attention block.  No gradient w.r.t. the exit input
    x (frozen backbone)."""
    grads = {}
    dy, dg_f = rmsnorm_backward(dz, act["yhat"], act["r_y"], params["g_f"])
    grads["g_f"] = dg_f
    if arch in MLP_BODY:
        M, A, B, u = act["M"], act["A"], act["B"], act["u"]
        grads["w_down"] = dy.T @ M                          # dW_down = dy^T M
        dM = dy @ params["w_down"]
        dA = dM * B * silu_grad(A)
        dB = dM * silu(A)
        grads["w_gate"] = dA.T @ u
        grads["w_up"] = dB.T @ u
        du = dA @ params["w_gate"] + dB @ params["w_up"]
        # u = g_a * xhat  =>  dg_a = sum_t du_t * xhat_t; no dx (frozen backbone)
        grads["g_a"] = np.sum(du * act["xhat"], axis=0)
    if arch == "layer":
        # through the MLP's pre-norm and residual into x1, then the attention block
        dxn, _ = rmsnorm_backward(du, act["xhat"], act["r_x"], params["g_a"])
        dx1 = dy + dxn
        grads.update(_attention_block_backward(params, act, dx1))
    return grads


def _attention_block_backward(params: dict, act: dict, dx1: np.ndarray) -> dict:
    """Gradients of x1 = x + W_o attn(...) w.r.t. g_att, W_q, W_k, W_v, W_o
    given dx1 (no gradient w.r.t. x: frozen backbone)."""
    N = dx1.shape[0]
    q, k, v = act["q"], act["k"], act["v"]
    grads = {"w_o": dx1.T @ act["o"]}                               # dW_o = dx1^T o
    do = (dx1 @ params["w_o"]).reshape(q.shape)
    dq, dk, dv = attention_backward(q, k, v, act["P"], do, act["T"])
    # RoPE is a rotation: its backward rotates by the opposite angle
    dq = rope(dq, -act["pos"], act["theta"]).reshape(N, -1)
    dk = rope(dk, -act["pos"], act["theta"]).reshape(N, -1)
    dv = dv.reshape(N, -1)
    u1 = act["u1"]
    grads["w_q"] = dq.T @ u1
    grads["w_k"] = dk.T @ u1
    grads["w_v"] = dv.T @ u1
    du1 = dq @ params["w_q"] + dk @ params["w_k"] + dv @ params["w_v"]
    grads["g_att"] = np.sum(du1 * act["xh1"], axis=0)
    return grads


def tune_step(arch: str, params_list, hidden_list, targets, exit_weights, eps: float,
              valid_count: int | None = None, attn: dict | None = None):
    """All exits of one step: exits are independent.

    Returns (losses [E] (unweighted L_i), grads list, stats list).
    """
    E = len(params_list)
    if len(hidden_list) != E or len(exit_weights) != E:
        raise ValueError("params, hidden and exit_weights must have one entry per exit")
    losses, grads, stats = [], [], []
    for i in range(E):
        r = exit_loss_and_grads(arch, params_list[i], hidden_list[i], targets,
                                float(exit_weights[i]), eps, valid_count, attn=attn)
        losses.append(r.loss)
        grads.append(r.grads)
        stats.append(r.stats)
    return np.array(losses), grads, stats


def exit_infer(arch: str, params_list, hidden_list, threshold: float, eps: float,
               attn: dict | None = None):
    """Confidence-based early exit at inference (§3 "Inference"):
    per exit the greedy token (argmax) and confidence (max softmax prob); a
    token exits at the first exit whose confidence reaches the threshold
    (threshold 1 disables early exits).  Returns (argmax [E,N],
    conf [E,N], first_exit [N], -1 = no early exit)."""
    am, cf = [], []
    for p, x in zip(params_list, hidden_list):
        S = exit_forward(arch, p, x, eps, attn)["S"]
        st = lm_loss_stats(S, np.full(S.shape[0], IGNORE_INDEX))
        am.append(st["argmax"])
        cf.append(st["conf"])
    am, cf = np.array(am), np.array(cf)
    first = np.full(cf.shape[1], -1, dtype=np.int64)
    for t in range(cf.shape[1]):
        for i in range(cf.shape[0]):
            if cf[i, t] >= threshold:
                first[t] = i
                break
    return am, cf, first


# ----------------------------------------------------------------------------
# optimizer (state for exits only; Adam constants)
# ----------------------------------------------------------------------------

def adam_update(theta, grad, m, v, lr, beta1, beta2, eps, weight_decay, step,
                grad_scale=1.0):
    """Kingma & Ba Adam with bias correction, eps outside the sqrt (A14).

    Returns new (theta, m, v).  ``step`` is the 1-based step count t.
    """
    g = grad_scale * grad
    m = beta1 * m + (1.0 - beta1) * g
    v = beta2 * v + (1.0 - beta2) * g * g
    mhat = m / (1.0 - beta1 ** step)
    vhat = v / (1.0 - beta2 ** step)
    theta = theta - lr * mhat / (np.sqrt(vhat) + eps) - lr * weight_decay * theta
    return theta, m, v


def sgd_update(theta, grad, buf, lr, momentum, grad_scale=1.0):
    """theta <- theta - lr * b with b = momentum * b + g (b = g when momentum is 0)."""
    g = grad_scale * grad
    buf = momentum * buf + g if buf is not None else g
    return theta - lr * buf, buf


def lr_at(it: int, total: int, warmup_frac: float = 0.01, lr_max: float = 1e-4,
          lr_min: float = 1e-5) -> float:
    """Linear warmup 0 -> lr_max over ceil(warmup_frac*total) iterations, then
    linear decay to lr_min at ``total`` (ramp origin 0 is A14)."""
    if total < 1 or it < 0 or it > total:
        raise ValueError("iteration out of range")
    w = int(math.ceil(warmup_frac * total))
    if w > 0 and it <= w:
        return lr_max * it / w
    if total == w:
        return lr_max
    return lr_max - (lr_max - lr_min) * (it - w) / (total - w)


def token_budget(batch: int = 16, seq: int = 2048, iters: int = 40000) -> int:
    """16 x 2048 x 4e4 tokens."""
    return batch * seq * iters


# ----------------------------------------------------------------------------
# Copy initialisation
# ----------------------------------------------------------------------------

def init_copy(arch: str, backbone: dict, after_layer: int) -> dict:
    """Exit parameters copied from the backbone (deep copies).

    backbone: ``final_norm`` [h], ``w_out`` [V,h], ``layers``: list of dicts with
    ``mlp_norm`` [h] (pre-MLP norm gain), ``w_gate``, ``w_up``, ``w_down``.
    Embedding/Norm copy the final-exit layer's modules; MLP copies the
    MLP of the same layer plus its pre-MLP norm gain (A10); Layer copies
    "the last Transformer layer of the original LLM" whatever the exit's
    position -- its attention (``g_att``, ``w_q``, ``w_k``, ``w_v``, ``w_o``)
    and MLP (``mlp_norm`` -> g_a, ``w_gate``, ``w_up``, ``w_down``).
    """
    if arch not in ARCHS:
        raise ValueError(f"unknown arch {arch!r}")
    if backbone.get("w_out") is None:
        raise LookupError("structure error: backbone has no output embedding")
    p = {"w_out": np.array(backbone["w_out"], copy=True)}
    if arch != "embedding":
        if backbone.get("final_norm") is None:
            raise LookupError("structure error: backbone has no final norm")
        p["g_f"] = np.array(backbone["final_norm"], copy=True)
    if arch == "mlp":
        layers = backbone.get("layers") or []
        if not (1 <= after_layer <= len(layers)):
            raise LookupError("structure error: no backbone layer to copy the MLP from")
        L = layers[after_layer - 1]
        for k_exit, k_bb in (("g_a", "mlp_norm"), ("w_gate", "w_gate"),
                             ("w_up", "w_up"), ("w_down", "w_down")):
            if L.get(k_bb) is None:
                raise LookupError(f"structure error: layer {after_layer} has no {k_bb}")
            p[k_exit] = np.array(L[k_bb], copy=True)
    if arch == "layer":
        layers = backbone.get("layers") or []
        if not layers or layers[-1] is None:
            raise LookupError("structure error: backbone has no last layer to copy")
        L = layers[-1]
        for k_exit, k_bb in (("g_att", "g_att"), ("w_q", "w_q"), ("w_k", "w_k"), ("w_v", "w_v"),
                             ("w_o", "w_o"), ("g_a", "mlp_norm"), ("w_gate", "w_gate"),
                             ("w_up", "w_up"), ("w_down", "w_down")):
            if L.get(k_bb) is None:
                raise LookupError(f"structure error: last layer has no {k_bb}")
            p[k_exit] = np.array(L[k_bb], copy=True)
    return p


def original_final_logits(backbone: dict, h_last: np.ndarray, eps: float) -> np.ndarray:
    """The original LLM's output layer on the last hidden state: final norm then
    output embedding ("optional layer normalization module, followed by a
    large output embedding matrix")."""
    g = backbone["final_norm"]
    r = 1.0 / np.sqrt(np.mean(h_last * h_last, axis=-1) + eps)
    return (g[None, :] * (h_last * r[:, None])) @ backbone["w_out"].T


# ----------------------------------------------------------------------------
# Frozen backbone partial forward (NEXT #3; §2.2 "Computational
# efficiency": "the partial forward pass of the Transformer backbone up to the
# hidden states connected to the last early exit")
# ----------------------------------------------------------------------------

def rope(x: np.ndarray, positions: np.ndarray, theta: float = 10000.0) -> np.ndarray:
    """Rotary position embedding, Llama "rotate-half" convention, applied to
    x [N, heads, d]: for i < d/2, angle_i(t) = t * theta^(-2i/d);
    out_i = x_i cos - x_{i+d/2} sin, out_{i+d/2} = x_{i+d/2} cos + x_i sin."""
    d = x.shape[-1]
    half = d // 2
    inv = theta ** (-np.arange(half, dtype=np.float64) * 2.0 / d)
    ang = positions.astype(np.float64)[:, None] * inv[None, :]          # [N, d/2]
    c, s = np.cos(ang)[:, None, :], np.sin(ang)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


def causal_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, seq_len: int) -> np.ndarray:
    """softmax(q k^T / sqrt(d) + causal mask) v within each sequence of
    seq_len consecutive rows; GQA: query head j uses kv head j // (Hq/Hkv).
    q [N, Hq, d], k, v [N, Hkv, d] -> [N, Hq, d]."""
    N, Hq, d = q.shape
    Hkv = k.shape[1]
    g = Hq // Hkv
    out = np.zeros_like(q)
    mask = np.triu(np.ones((seq_len, seq_len), dtype=bool), 1)
    for b in range(N // seq_len):
        rs = slice(b * seq_len, (b + 1) * seq_len)
        for j in range(Hq):
            S = q[rs, j, :] @ k[rs, j // g, :].T / math.sqrt(d)
            S = np.where(mask, -np.inf, S)
            S = S - S.max(axis=1, keepdims=True)
            P = np.exp(S)
            P /= P.sum(axis=1, keepdims=True)
            out[rs, j, :] = P @ v[rs, j // g, :]
    return out


def llama_layer_forward(layer: dict, x: np.ndarray, seq_len: int, n_heads: int, n_kv: int,
                        eps: float, theta: float = 10000.0) -> np.ndarray:
    """One pre-norm Llama-2 decoder layer (the backbone the paper tunes on,
    P:356-358; "residual structure with pre-normalization"):
    x += Wo attn(RoPE(Wq u), RoPE(Wk u), Wv u), u = RMSNorm(x; g_att);
    x += W_down(silu(W_gate u') * W_up u'), u' = RMSNorm(x; g_mlp)."""
    N, h = x.shape
    d = h // n_heads
    pos = np.arange(N) % seq_len
    u, _, _ = rmsnorm(x, layer["g_att"], eps)
    q = (u @ layer["w_q"].T).reshape(N, n_heads, d)
    k = (u @ layer["w_k"].T).reshape(N, n_kv, d)
    v = (u @ layer["w_v"].T).reshape(N, n_kv, d)
    q, k = rope(q, pos, theta), rope(k, pos, theta)
    o = causal_attention(q, k, v, seq_len).reshape(N, n_heads * d)
    x = x + o @ layer["w_o"].T
    u2, _, _ = rmsnorm(x, layer["g_mlp"], eps)
    x = x + (silu(u2 @ layer["w_gate"].T) * (u2 @ layer["w_up"].T)) @ layer["w_down"].T
    return x


def backbone_forward(layers, x0: np.ndarray, seq_len: int, n_heads: int, n_kv: int,
                     exit_after, eps: float, theta: float = 10000.0):
    """Runs layers 1..max(exit_after) only (the partial forward of P:260) and
    returns the hidden state after each requested layer (the exits' inputs)."""
    outs = {}
    x = x0
    last = max(exit_after)
    for l in range(1, last + 1):
        x = llama_layer_forward(layers[l - 1], x, seq_len, n_heads, n_kv, eps, theta)
        if l in exit_after:
            outs[l] = x.copy()
    return [outs[l] for l in exit_after]
