"""Property-based pins of the fp64 oracle over random small shapes (hypothesis):
what the mathematics fixes for every arch and shape, not just the fixed
shapes of test_oracle_pins.py.
  * softmax-CE gradient rows sum to zero, so sum_v dW_out[v, :] = 0 (P4);
  * a central-difference directional derivative along a random direction of
    ALL exit parameters equals <grad, direction> (P6 generalised);
  * token permutations leave the loss and the gradients unchanged for the
    token-independent archs (tokens are independent);
  * ignored targets (-1) contribute nothing: dropping those tokens changes
    neither loss nor gradients (A6)."""

import numpy as np
from hypothesis import given, settings, strategies as st

from oracle import ee_oracle as O

ARCHS = ("embedding", "norm", "mlp")


def _params(arch, h, V, F, rng, w=0.4):
    p = {"w_out": rng.normal(0, w, (V, h))}
    if arch != "embedding":
        p["g_f"] = 1.0 + 0.1 * rng.normal(size=h)
    if arch == "mlp":
        p["g_a"] = 1.0 + 0.1 * rng.normal(size=h)
        p["w_gate"] = rng.normal(0, w, (F, h))
        p["w_up"] = rng.normal(0, w, (F, h))
        p["w_down"] = rng.normal(0, w, (h, F))
    return p


shape = st.tuples(st.sampled_from(ARCHS), st.integers(2, 9), st.integers(2, 13),
                  st.integers(1, 7), st.integers(1, 11), st.integers(0, 2**31 - 1))


@settings(max_examples=40, deadline=None)
@given(shape)
def test_dW_out_columns_sum_to_zero(s):
    arch, h, V, F, N, seed = s
    rng = np.random.default_rng(seed)
    p = _params(arch, h, V, F, rng)
    x = rng.normal(size=(N, h))
    y = rng.integers(-1, V, N)
    r = O.exit_loss_and_grads(arch, p, x, y, 0.7, 1e-5)
    scale = np.abs(r.grads["w_out"]).sum() + 1e-300
    assert np.abs(r.grads["w_out"].sum(axis=0)).max() <= 1e-12 * max(1.0, scale)


@settings(max_examples=25, deadline=None)
@given(shape)
def test_directional_derivative_matches_gradient(s):
    arch, h, V, F, N, seed = s
    rng = np.random.default_rng(seed)
    p = _params(arch, h, V, F, rng)
    x = rng.normal(size=(N, h))
    y = rng.integers(0, V, N)
    r = O.exit_loss_and_grads(arch, p, x, y, 1.0, 1e-5)
    d = {k: rng.normal(size=v.shape) for k, v in p.items()}
    eps = 1e-5

    def loss_at(t):
        q = {k: p[k] + t * d[k] for k in p}
        return O.exit_loss_and_grads(arch, q, x, y, 1.0, 1e-5).loss
    fd = (loss_at(eps) - loss_at(-eps)) / (2 * eps)
    an = sum(float(np.sum(r.grads[k] * d[k])) for k in p)
    assert abs(fd - an) <= 1e-6 * max(1.0, abs(an))


@settings(max_examples=25, deadline=None)
@given(shape)
def test_token_permutation_invariance(s):
    arch, h, V, F, N, seed = s
    rng = np.random.default_rng(seed)
    p = _params(arch, h, V, F, rng)
    x = rng.normal(size=(N, h))
    y = rng.integers(-1, V, N)
    perm = rng.permutation(N)
    a = O.exit_loss_and_grads(arch, p, x, y, 1.0, 1e-5)
    b = O.exit_loss_and_grads(arch, p, x[perm], y[perm], 1.0, 1e-5)
    assert abs(a.loss - b.loss) <= 1e-12 * max(1.0, abs(a.loss))
    for k in a.grads:
        np.testing.assert_allclose(a.grads[k], b.grads[k], rtol=1e-10, atol=1e-13)


@settings(max_examples=25, deadline=None)
@given(shape)
def test_ignored_tokens_contribute_nothing(s):
    arch, h, V, F, N, seed = s
    rng = np.random.default_rng(seed)
    p = _params(arch, h, V, F, rng)
    x = rng.normal(size=(N + 3, h))
    y = rng.integers(0, V, N + 3)
    y[-3:] = -1                                      # three ignored tokens
    a = O.exit_loss_and_grads(arch, p, x, y, 1.0, 1e-5)
    b = O.exit_loss_and_grads(arch, p, x[:-3], y[:-3], 1.0, 1e-5)
    assert abs(a.loss - b.loss) <= 1e-12 * max(1.0, abs(a.loss))
    for k in a.grads:
        np.testing.assert_allclose(a.grads[k], b.grads[k], rtol=1e-10, atol=1e-13)
