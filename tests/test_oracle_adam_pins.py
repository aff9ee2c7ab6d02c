"""Pins for the oracle's adapter update: bias-corrected
Adam (Kingma & Ba, ICLR 2015, Algorithm 1).  Closed forms
that a dropped bias correction, a swapped beta or a missing square root fail."""
import numpy as np


def test_spec_first_step_example(oracle_mod):
    """w = 1, g = 1, lr = 0.1, first step -> w = 1 - 0.1 / (1 + eps)."""
    th, m, v = oracle_mod.adam_step([1.0], [1.0], [0.0], [0.0], 1, 0.1)
    assert th[0] == 1.0 - 0.1 / (1.0 + 1e-8)
    assert abs(m[0] - 0.1) < 1e-16 and abs(v[0] - 0.001) < 1e-18


def test_zero_gradient_zero_state_is_identity(oracle_mod):
    th0 = np.linspace(-2, 3, 11)
    th, m, v = oracle_mod.adam_step(th0, np.zeros(11), np.zeros(11), np.zeros(11), 1, 0.5)
    np.testing.assert_array_equal(th, th0)
    np.testing.assert_array_equal(m, 0.0)
    np.testing.assert_array_equal(v, 0.0)


def test_constant_gradient_closed_form(oracle_mod):
    """For a constant gradient g the bias-corrected moments are exactly g and
    g^2 at every step, so theta_t = theta_0 - t lr g / (|g| + eps)."""
    g = np.array([0.5, -3.0, 1e-3, 7.0])
    th0 = np.array([1.0, 2.0, -1.0, 0.0])
    th, m, v = th0.copy(), np.zeros(4), np.zeros(4)
    lr, eps = 1e-2, 1e-8
    for t in range(1, 7):
        th, m, v = oracle_mod.adam_step(th, g, m, v, t, lr, eps=eps)
        np.testing.assert_allclose(th, th0 - t * lr * g / (np.abs(g) + eps), rtol=0, atol=1e-13)


def test_scale_invariance_and_unit_first_step(oracle_mod):
    """With eps = 0 Adam is invariant to a positive gradient scale, and the
    first step moves every coordinate by exactly lr * sign(g)."""
    rng = np.random.default_rng(5)
    g1, g2 = rng.normal(size=16), rng.normal(size=16)
    th0 = rng.normal(size=16)
    a1 = oracle_mod.adam_step(th0, g1, np.zeros(16), np.zeros(16), 1, 0.25, eps=0.0)
    np.testing.assert_allclose(a1[0], th0 - 0.25 * np.sign(g1), rtol=0, atol=1e-15)
    a2 = oracle_mod.adam_step(a1[0], g2, a1[1], a1[2], 2, 0.25, eps=0.0)
    b1 = oracle_mod.adam_step(th0, 7.0 * g1, np.zeros(16), np.zeros(16), 1, 0.25, eps=0.0)
    b2 = oracle_mod.adam_step(b1[0], 7.0 * g2, b1[1], b1[2], 2, 0.25, eps=0.0)
    np.testing.assert_allclose(b2[0], a2[0], rtol=0, atol=1e-14)


def test_three_step_trajectory_by_hand(oracle_mod):
    """a 3-step scalar trajectory, the moments unrolled by hand:
    m_3 = (1-b1)(b1^2 g1 + b1 g2 + g3), v_3 = (1-b2)(b2^2 g1^2 + b2 g2^2 + g3^2)."""
    b1, b2, lr, eps = 0.9, 0.999, 1e-3, 1e-8
    gs = [0.3, -0.7, 1.1]
    th, m, v = np.array([0.5]), np.zeros(1), np.zeros(1)
    for t, g in enumerate(gs, 1):
        th, m, v = oracle_mod.adam_step(th, [g], m, v, t, lr, b1, b2, eps)
    m3 = (1 - b1) * (b1 ** 2 * gs[0] + b1 * gs[1] + gs[2])
    v3 = (1 - b2) * (b2 ** 2 * gs[0] ** 2 + b2 * gs[1] ** 2 + gs[2] ** 2)
    assert abs(m[0] - m3) < 1e-15 and abs(v[0] - v3) < 1e-15
