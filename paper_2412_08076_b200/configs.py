"""Seeded synthetic inputs for the five BASELINE.json configs.

The reference has no dataset: every config is a seeded draw, resolved as
SURVEY.md §8(d) / Appendix B prescribe.  The weight / symbol generators are
random-init PyTorch networks (the "meta-network" side, host PyTorch as in
the north star); they only produce arrays, which the GPU path and the CPU
oracle then consume identically.

  cfg1  Richardson(8), 63^2, theta=pi/6, eps=1e-2, f ~ N(0,1) seed 0,
        Chebyshev weights on [lambda_min50, 1.01 lambda_max50] from 50-step
        power iterations; to 1e-6.
  cfg2  NAG(16), 64 x 255^2, (lg eps, theta) random, random-init GELU MLP
        3x64 -> 32 (omega = softplus, alpha = sigmoid), 200 outer; f64 and f32.
  cfg3  Jacobi Richardson(32), 8 x 1023^2, Leja-ordered Chebyshev of the
        scaled operator (lambda_max: symbol maximum; lambda_min: small-grid
        eigenvalues extrapolated in h^2, x0.9); to 1e-6.
  cfg4  FNS: 4 x 1023^2, eps=1e-3, symbol from a random-init 4-layer conv net
        on the sine-frequency grid (x0.01), M = 8 smoothing steps omega=0.5;
        100 alternations.
  cfg5  Helmholtz, 4 right-hand sides on 1023^2 (k h = 2 pi/10, sponge),
        Gaussian source + N(0, 0.1^2) noise, NAG(16) weights from a
        random-init MLP on k re-centred at 0.8/(8 n^2); V-cycle (coarsest 16)
        inside FGMRES(20), 5 restarts = 100 preconditioner applications.
"""
from __future__ import annotations

import numpy as np
import torch

from .problems import AnisotropicProblem, HelmholtzProblem, anisotropic_stencil
from .schedules import (WeightSchedule, chebyshev_weights, leja_order, stencil_lambda_min,
                        stencil_symbol_bounds)

ANISOTROPIC_BOUNDS = np.array([[-6.0, 0.0], [0.0, np.pi]])  # metanet.py:24 (lg eps, theta)


# ------------------------------------------------------------------ helpers
def stencil_matvec_host(c, s, x):
    """y = A x for a constant 9-point stencil on an s x s grid (host NumPy,
    CSR summation order; used only for the cfg1 power-iteration recipe)."""
    X = np.zeros((s + 2, s + 2))
    X[1:-1, 1:-1] = x.reshape(s, s)
    y = np.zeros((s, s))
    q = 0
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            y = y + c[q] * X[1 + dx:1 + dx + s, 1 + dy:1 + dy + s]
            q += 1
    return y.reshape(-1)


def power_bounds(matvec, n, steps=50, seed=0, shift=1.01):
    """cfg1 recipe (spectral.py:31-82 with a fixed step count): Rayleigh
    quotient after `steps` power steps, then `steps` shifted steps with
    sigma = shift * lambda_max."""
    def run(mv):
        rng = np.random.default_rng(seed)
        x = rng.standard_normal(n)
        x /= np.linalg.norm(x)
        lam = 0.0
        for _ in range(steps):
            y = mv(x)
            lam = float(np.real(np.vdot(x, y)))
            x = y / np.linalg.norm(y)
        return lam
    lmax = run(matvec)
    sigma = shift * lmax
    lmin = sigma - run(lambda x: sigma * x - matvec(x))
    return lmax, lmin


class _MLP(torch.nn.Module):
    """Random-init GELU MLP, output layer scaled like MetaNet.create
    (metanet.py:47-66: weights x0.01, bias -2)."""

    def __init__(self, din, dout, hidden=64, layers=3, out_bias=-2.0):
        super().__init__()
        dims = [din] + [hidden] * layers
        self.body = torch.nn.ModuleList(torch.nn.Linear(a, b) for a, b in zip(dims, dims[1:]))
        self.out = torch.nn.Linear(hidden, dout)
        with torch.no_grad():
            self.out.weight.mul_(0.01)
            self.out.bias.fill_(out_bias)

    def forward(self, x):
        for lin in self.body:
            x = torch.nn.functional.gelu(lin(x))
        return self.out(x)


# ------------------------------------------------------------------ configs
def cfg1():
    p = AnisotropicProblem(1e-2, np.pi / 6, 64)
    c = anisotropic_stencil(p)
    s = p.n - 1
    f = np.random.default_rng(0).standard_normal(s * s)
    lmax, lmin = power_bounds(lambda x: stencil_matvec_host(c, s, x), s * s)
    omega = chebyshev_weights(1.01 * lmax, lmin, 8)
    return dict(problem=p, f=f, schedule=WeightSchedule(omega=omega), tol=1e-6,
                lmax50=lmax, lmin50=lmin)


def cfg2(batch=64, n=256, m=16, outer=200):
    rng = np.random.default_rng(2)
    probs, F = [], []
    for _ in range(batch):
        theta = rng.uniform(0.0, np.pi)
        lg = rng.uniform(-5.0, 0.0)
        probs.append(AnisotropicProblem(10.0 ** lg, theta, n))
        F.append(rng.standard_normal((n - 1) ** 2))
    torch.manual_seed(2)
    net = _MLP(2, 2 * m).double()
    mu = torch.tensor([[np.log10(p.epsilon), p.theta] for p in probs], dtype=torch.float64)
    lo, hi = torch.tensor(ANISOTROPIC_BOUNDS[:, 0]), torch.tensor(ANISOTROPIC_BOUNDS[:, 1])
    with torch.no_grad():
        raw = net(2.0 * (mu - lo) / (hi - lo) - 1.0).numpy()   # metanet.py:86-88 normalisation
    omega = np.log1p(np.exp(raw[:, :m]))                     # softplus (metanet.py:100)
    alpha = 1.0 / (1.0 + np.exp(-raw[:, m:]))                # sigmoid (metanet.py:101-102)
    scheds = [WeightSchedule(omega=omega[b], alpha=alpha[b], variant="nag") for b in range(batch)]
    return dict(problems=probs, F=np.stack(F), schedules=scheds, outer=outer, m=m)


def cfg3(first=0, count=8, n=1024, m=32, seed=3):
    rng = np.random.default_rng(seed)
    probs, F, scheds, scales = [], [], [], []
    for b in range(first + count):
        theta = rng.uniform(0.0, np.pi)
        eps = 10.0 ** rng.uniform(-4.0, 0.0)
        f = rng.standard_normal((n - 1) ** 2)
        if b < first:
            continue
        p = AnisotropicProblem(float(eps), float(theta), n)
        c = anisotropic_stencil(p)
        sc = (2.0 / 3.0) / c[4]                  # weighted Jacobi, relax 2/3 (precond.py:71-77)
        lmax = stencil_symbol_bounds(c, n)[0]
        lmin = stencil_lambda_min(c, n)
        probs.append(p)
        F.append(f)
        scheds.append(WeightSchedule(omega=leja_order(chebyshev_weights(sc * lmax, sc * lmin, m))))
        scales.append(sc)
    return dict(problems=probs, F=np.stack(F), schedules=scheds, scales=np.array(scales), m=m)


def nag_sweep(first=0, count=8, n=1024, m=16):
    """The north-star batched NAG(16) sweep at 1023^2: cfg3's systems
    (default_rng(3)), NAG weights from cfg2's random-init MLP (same network
    and seed, torch.manual_seed(2)) evaluated at each system's (lg eps, theta)."""
    c3 = cfg3(first=first, count=count, n=n)
    probs = c3["problems"]
    torch.manual_seed(2)
    net = _MLP(2, 2 * m).double()
    mu = torch.tensor([[np.log10(p.epsilon), p.theta] for p in probs], dtype=torch.float64)
    lo, hi = torch.tensor(ANISOTROPIC_BOUNDS[:, 0]), torch.tensor(ANISOTROPIC_BOUNDS[:, 1])
    with torch.no_grad():
        raw = net(2.0 * (mu - lo) / (hi - lo) - 1.0).numpy()
    omega = np.log1p(np.exp(raw[:, :m]))
    alpha = 1.0 / (1.0 + np.exp(-raw[:, m:]))
    scheds = [WeightSchedule(omega=omega[b], alpha=alpha[b], variant="nag")
              for b in range(len(probs))]
    return dict(problems=probs, F=c3["F"], schedules=scheds, m=m)


def fns_symbol(theta, eps, n, seed=4, scale=0.01, device="cuda"):
    """Random-init 4-layer conv net on the (n-1)^2 sine-frequency grid with
    channels (theta, eps, p/n, q/n) -> real symbol (fns.py:36: real), x scale."""
    torch.manual_seed(seed)
    net = torch.nn.Sequential(
        torch.nn.Conv2d(4, 16, 3, padding=1), torch.nn.GELU(),
        torch.nn.Conv2d(16, 16, 3, padding=1), torch.nn.GELU(),
        torch.nn.Conv2d(16, 16, 3, padding=1), torch.nn.GELU(),
        torch.nn.Conv2d(16, 1, 3, padding=1)).double().to(device)
    s = n - 1
    pq = torch.arange(1, n, dtype=torch.float64, device=device) / n
    P, Q = torch.meshgrid(pq, pq, indexing="ij")
    x = torch.stack([torch.full_like(P, theta), torch.full_like(P, eps), P, Q])[None]
    with torch.no_grad():
        lam = net(x)[0, 0] * scale
    return lam.reshape(s * s).contiguous()


def fns_symbol_portable(theta, eps, n, seed=4, scale=0.01):
    """cfg4's conv-net symbol evaluated on the CPU and rounded to float32
    (then widened back) as a NumPy array: the rounding absorbs last-bit
    differences between BLAS builds, so the full-size goldens
    (tests/golden/full_cfg4.npz) and the GPU test see the same bits on any
    machine (the test checks the sha256)."""
    lam = fns_symbol(theta, eps, n, seed=seed, scale=scale, device="cpu")
    return lam.float().double().numpy()


def cfg4(batch=4, n=1024, eps=1e-3, M=8, alternations=100, device="cuda"):
    rng = np.random.default_rng(4)
    probs, F = [], []
    for _ in range(batch):
        theta = rng.uniform(0.0, np.pi)
        probs.append(AnisotropicProblem(eps, float(theta), n))
        F.append(rng.standard_normal((n - 1) ** 2))
    lam = torch.stack([fns_symbol(p.theta, p.epsilon, n, device=device) for p in probs])
    return dict(problems=probs, F=np.stack(F), lam=lam, schedule=WeightSchedule(omega=np.full(8, 0.5)),
                M=M, alternations=alternations)


def cfg5(batch=4, n=1024, m=16, device="cuda"):
    rng = np.random.default_rng(5)
    hp = HelmholtzProblem(2 * np.pi * n / 10, n)   # k h = 2 pi / 10
    s = n - 1
    h = 1.0 / n
    x = np.arange(1, n) * h
    X, Y = np.meshgrid(x, x, indexing="ij")
    F = []
    for _ in range(batch):
        i0, j0 = rng.integers(1, n, size=2)
        sig = 4 * h
        bump = np.exp(-((X - i0 * h) ** 2 + (Y - j0 * h) ** 2) / (2 * sig ** 2))
        F.append((bump + rng.normal(0.0, 0.1, size=(s, s))).reshape(-1).astype(np.complex128))
    torch.manual_seed(5)
    net = _MLP(1, 2 * m, out_bias=0.0).double()
    with torch.no_grad():
        net.out.bias[m:] = -2.0                         # alpha ~ sigmoid(-2) ~ 0.12
        raw = net(torch.tensor([[hp.angular_frequency / (2 * np.pi * n)]], dtype=torch.float64))[0].numpy()
    omega = (0.8 / (8 * n * n)) * np.exp(raw[:m])       # log-omega mode re-centred
    alpha = 1.0 / (1.0 + np.exp(-raw[m:]))
    return dict(problem=hp, F=np.stack(F),
                schedule=WeightSchedule(omega=omega, alpha=alpha, variant="nag"),
                coarsest=16, restart=20, max_outer=5)
