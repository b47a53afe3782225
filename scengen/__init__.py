"""Seeded synthetic scenario generator -- the ONLY module shared by the oracle
and the CUDA path.  It holds none of the solver's arithmetic: it only draws
inputs (task lengths, channel gains, acceptance rates) and names the parameter
presets printed in the paper's Tables I and II.

Workload recipe (paper Sec. IV "Simulation Results"):
  * K tasks per scenario, users uniform over a disk of radius R = 400 m
    around the SBS, d_k = max(1 m, R*sqrt(U)) (uniform over the disk;
    DESIGN.md reading R3 -- the paper does not say how users are placed).
  * g_k = g0 * rho_k * d_k^-2 with rho_k ~ Exp(1) (Rayleigh power fading),
    g0 = 1e-3 ("-30 dBm" path-loss constant read as -30 dB, reading R2).
  * I_k uniform on {1..I_max}, I_max = 512 (Table II).
  * p_k = 0.2 W (Table II).
  * alpha ~ U[0.5, 0.9) per scenario (BASELINE.json configs[2]).

Counter-based, so any shard or sample of a config is generated independently
and bit-identically: draw c of scenario s under root seed r is
    u64(r, s, c) = mix(mix(r*PHI ^ SALT + s*PHI) + (c+1)*PHI)
with mix = splitmix64's finaliser and PHI = 0x9E3779B97F4A7C15 (all mod 2^64).
Draw order inside a scenario: c = 0 -> alpha; for task k: c = 1+3k -> I_k,
c = 2+3k -> distance, c = 3+3k -> fading.  U01 = (u >> 11) * 2^-53 in [0,1);
U01o = ((u >> 11) + 1) * 2^-53 in (0,1].
"""
from __future__ import annotations

import numpy as np

PHI = np.uint64(0x9E3779B97F4A7C15)
SALT = np.uint64(0xD1B54A32D192ED03)
M1 = np.uint64(0xBF58476D1CE4E5B9)
M2 = np.uint64(0x94D049BB133111EB)

# Table I: name -> (layers J, hidden h1, ffn h2)
MODELS = {
    "68M": (2, 768, 3072),
    "1.1B": (22, 2048, 5632),
    "7B": (32, 4096, 11008),
    "13B": (40, 5120, 13824),
}

# Table II and Sec. IV
TABLE2 = dict(
    c1_verify=2.08e-14,
    c2_verify=1.28e-2,
    c1_draft=4.11e-13,
    c2_draft=0.56e-3,
    bandwidth_hz=20e6,
    noise_w=10.0 ** ((-106.0 - 30.0) / 10.0),  # -106 dBm in W (reading R1)
    mem_capacity_bytes=16_000_000_000,  # "16 GB" read as SI (reading A9)
    O_max=2048,
    I_max=512,
    tx_power_w=0.2,
    g0=1e-3,
    radius_m=400.0,
)


def _mix(z):
    z = (z ^ (z >> np.uint64(30))) * M1
    z = (z ^ (z >> np.uint64(27))) * M2
    return z ^ (z >> np.uint64(31))


def u64(root: int, s, c):
    """Counter-based 64-bit draw for scenario index array `s`, counter `c`."""
    with np.errstate(over="ignore"):
        s = np.asarray(s, dtype=np.uint64)
        c = np.asarray(c, dtype=np.uint64)
        key = _mix(np.uint64(root) * PHI ^ SALT + s * PHI)
        return _mix(key + (c + np.uint64(1)) * PHI)


def _u01(u):
    return (u >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def _u01_open0(u):
    return ((u >> np.uint64(11)).astype(np.float64) + 1.0) * (2.0 ** -53)


def params(pair: str = "68M-7B", K: int = 128, gamma_min: int = 1, gamma_max: int = 16,
           **overrides) -> dict:
    """Plain-dict solver parameters (Tables I/II defaults).  Each side of the
    parity check marshals this into its own struct."""
    d, v = pair.split("-")
    p = dict(TABLE2)
    p.update(draft=MODELS[d], verify=MODELS[v], K=K, gamma_min=gamma_min,
             gamma_max=gamma_max, lambda_bits=0.0, downlink_s=0.0, precision=0)
    for k in ("I_max", "tx_power_w", "g0", "radius_m"):
        p.pop(k)
    p.update(overrides)
    return p


def generate(root: int, K: int, s0: int, s1: int, I_max: int = 512,
             alpha_lo: float = 0.5, alpha_hi: float = 0.9, tx_power_w: float = 0.2,
             g0: float = 1e-3, radius_m: float = 400.0, chunk: int = 1 << 15) -> dict:
    """Scenarios s0..s1-1 of root seed `root` (SoA numpy arrays)."""
    if s1 - s0 > chunk:
        parts = [generate(root, K, a, min(a + chunk, s1), I_max, alpha_lo, alpha_hi, tx_power_w, g0,
                          radius_m, chunk) for a in range(s0, s1, chunk)]
        return {k: (np.concatenate([q[k] for q in parts]) if parts[0][k] is not None else None)
                for k in parts[0]}
    n = s1 - s0
    s = np.arange(s0, s1, dtype=np.uint64)[:, None]
    k = np.arange(K, dtype=np.uint64)[None, :]
    alpha = alpha_lo + (alpha_hi - alpha_lo) * _u01(u64(root, s[:, 0], 0))
    I = (1 + np.floor(I_max * _u01(u64(root, s, 1 + 3 * k)))).astype(np.int32)
    dist = np.maximum(1.0, radius_m * np.sqrt(_u01_open0(u64(root, s, 2 + 3 * k))))
    rho = -np.log(_u01_open0(u64(root, s, 3 + 3 * k)))
    g = g0 * rho / (dist * dist)
    p = np.full((n, K), tx_power_w, dtype=np.float64)
    return dict(I=np.ascontiguousarray(I), p=p, g=np.ascontiguousarray(g),
                alpha=np.ascontiguousarray(alpha), coeffs=None)


def output_lengths(root: int, K: int, s0: int, s1: int, O_max: int = 2048) -> np.ndarray:
    """Actual output lengths O_k uniform on {1..O_max}, counter c = 1 + 3K + k
    (after the task draws), for the actual-output evaluation."""
    s = np.arange(s0, s1, dtype=np.uint64)[:, None]
    k = np.arange(K, dtype=np.uint64)[None, :]
    return np.ascontiguousarray((1 + np.floor(O_max * _u01(u64(root, s, 1 + 3 * K + k)))).astype(np.int32))


# ---------------------------------------------------------------- configs
# SURVEY.md Sec. 8(d) table; BASELINE.json "configs".
GOLDEN_C1 = dict(I=[512, 37, 255, 100], g=[1e-8, 4e-9, 2.5e-8, 1e-9], alpha=0.8)


def config(name: str, s0: int = 0, s1: int | None = None, pair: str | None = None):
    """Return (params, scenarios, n_total) for BASELINE configs C1..C5.

    C1  K=4, gamma 0..4, the fixed golden instance (scenario 0) followed by
        seeded K=4 scenarios (n_total = 1001).
    C2  K=64, gamma 1..8, (1.1B,7B), alpha=0.8, three scenarios with the draft
        node's c1,c2 scaled by 1/4, 1, 4 (heterogeneous node speeds).
    C3  1e5 x K=32, gamma 1..8.     C4  1e6 x K=128, gamma 1..16.
    C5k 1e4 x K=k (k in 256,512,1024), gamma 1..16.
    """
    if name == "C1":
        pr = params(pair or "68M-7B", K=4, gamma_min=0, gamma_max=4)
        n_total = 1001
        s1 = n_total if s1 is None else s1
        sc = generate(1, 4, s0, s1)
        if s0 == 0 and s1 > 0:
            sc["I"][0] = GOLDEN_C1["I"]
            sc["g"][0] = GOLDEN_C1["g"]
            sc["alpha"][0] = GOLDEN_C1["alpha"]
        return pr, sc, n_total
    if name == "C2":
        pr = params(pair or "1.1B-7B", K=64, gamma_min=1, gamma_max=8)
        n_total = 3
        s1 = n_total if s1 is None else s1
        sc = generate(2, 64, s0, s1)
        sc["alpha"][:] = 0.8
        scale = np.array([0.25, 1.0, 4.0])[s0:s1]
        co = np.empty((s1 - s0, 4))
        co[:, 0] = pr["c1_draft"] * scale
        co[:, 1] = pr["c2_draft"] * scale
        co[:, 2] = pr["c1_verify"]
        co[:, 3] = pr["c2_verify"]
        sc["coeffs"] = co
        return pr, sc, n_total
    if name == "C3":
        pr = params(pair or "68M-7B", K=32, gamma_min=1, gamma_max=8)
        n_total = 100_000
        s1 = n_total if s1 is None else s1
        return pr, generate(3, 32, s0, s1), n_total
    if name == "C4":
        pr = params(pair or "68M-7B", K=128, gamma_min=1, gamma_max=16)
        n_total = 1_000_000
        s1 = n_total if s1 is None else s1
        return pr, generate(4, 128, s0, s1), n_total
    if name.startswith("C5"):
        K = int(name[2:] or 256)
        pr = params(pair or "68M-7B", K=K, gamma_min=1, gamma_max=16)
        n_total = 10_000
        s1 = n_total if s1 is None else s1
        return pr, generate(5, K, s0, s1), n_total
    raise ValueError(name)
