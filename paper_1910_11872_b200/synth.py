"""Seeded synthetic complex fringe stacks (the inputs both the CUDA path and the oracle see).

This module holds only the *signal model* of Eq.(1) and the phase phantoms of
DESIGN.md §4 — none of the estimator's arithmetic.  It is the one module shared by the
tests, the bench and (through the tests) the oracle: the oracle always consumes the exact
complex64 bytes produced here, copied to the host.

    Γ_t(x,y) = A·exp(j(ω_cx·x + ω_cy·y + φ_t(x,y))) + η_t(x,y)        Eq.(1)

with A = 1, carrier (f_x, f_y) = (1/16, 1/8) cycles/px, η circular complex Gaussian with
E|η|² = 10^{-SNR/10} (SNR over the total complex noise variance, DESIGN.md [R9]).  Noise of
frame t is drawn from a torch generator keyed by (seed, global frame index t), so a frame's
bytes do not depend on which rank (or which shard) generates it on a given device type.
"""

from __future__ import annotations

import math
from dataclasses import dataclass, field

import torch

CARRIER_FX = 1.0 / 16.0
CARRIER_FY = 1.0 / 8.0

# Diffusion phantom constants: pixel pitch 9.1 µm, D of NaCl-water
# (assumed; the paper does not give it), Φ0 = 20 rad at t1 = 60 s.
PIXEL_PITCH_M = 9.1e-6
DIFFUSION_D = 1.5e-9
DIFF_PHI0 = 20.0
DIFF_T1 = 60.0


def _grid(H, W, device):
    y = torch.arange(H, dtype=torch.float64, device=device)[:, None]
    x = torch.arange(W, dtype=torch.float64, device=device)[None, :]
    return y, x


def carrier_phase(H, W, device="cpu", fx=CARRIER_FX, fy=CARRIER_FY):
    y, x = _grid(H, W, device)
    return 2.0 * math.pi * (fx * x + fy * y)


def gaussian(H, W, amp, x0, y0, sigma, device="cpu"):
    y, x = _grid(H, W, device)
    return amp * torch.exp(-((x - x0) ** 2 + (y - y0) ** 2) / (2.0 * sigma * sigma))


def phase_c1(H=256, W=256, device="cpu"):
    """C1: centred Gaussian, 1.0 rad, σ = 100 px (max|∇²φ| = 2e-4 rad/px²)."""
    return gaussian(H, W, 1.0, (W - 1) / 2.0, (H - 1) / 2.0, 100.0, device)


def phase_plane(H, W, gx=0.3, gy=-0.7, c=0.4, device="cpu"):
    y, x = _grid(H, W, device)
    return gx * x + gy * y + c


def phase_c2_flow(H=512, W=512, device="cpu"):
    """C2 flow frame: three Gaussian lobes, ≈22 rad peak-to-valley (SPEC S:L363 style)."""
    s = H / 512.0
    return (gaussian(H, W, 14.0, 180 * s, 200 * s, 60 * s, device)
            - gaussian(H, W, 8.0, 340 * s, 300 * s, 70 * s, device)
            + gaussian(H, W, 6.0, 300 * s, 140 * s, 50 * s, device))


def phase_diffusion(H, W, t_s, device="cpu"):
    """Diffusion phantom: φ ∝ ∂c/∂y of the free-diffusion step solution of Eq.(16)
    (c = (c0/2)erfc(s/2√(Dt)), ∂c/∂s ∝ exp(-s²/4Dt)/√t), mapped to phase by Eq.(17)
    (phase ∝ ∂n/∂x).  Interface at the frame's middle row."""
    y, x = _grid(H, W, device)
    s = (y - H / 2.0) * PIXEL_PITCH_M
    prof = DIFF_PHI0 * math.sqrt(DIFF_T1 / t_s) * torch.exp(-(s * s) / (4.0 * DIFFUSION_D * t_s))
    return prof.expand(H, W)


@dataclass
class Workload:
    name: str
    H: int
    W: int
    T: int
    window_len: int
    snr_db: float | None
    seed: int
    kind: str                      # "c1", "plane", "c2", "diffusion"
    times: list = field(default_factory=list)   # diffusion frame times (s); frame 0 = reference

    def phase(self, t: int, device="cpu"):
        """Flow phase φ_t of frame t (frame 0 of a stack is the reference: φ = 0)."""
        H, W = self.H, self.W
        if self.kind == "c1":
            return phase_c1(H, W, device)
        if self.kind == "plane":
            return phase_plane(H, W, device=device)
        if self.kind == "c2":
            return torch.zeros(H, W, dtype=torch.float64, device=device) if t == 0 \
                else phase_c2_flow(H, W, device)
        if self.kind == "diffusion":
            if t == 0:
                return torch.zeros(H, W, dtype=torch.float64, device=device)
            return phase_diffusion(H, W, self.time_of(t), device)
        raise ValueError(self.kind)

    def time_of(self, t: int) -> float:
        """Diffusion time of global flow frame t ≥ 1.  Frame indices beyond the schedule
        (multi-GPU weak scaling: rank r owns flow frames r·(T−1)+1 … (r+1)·(T−1)) repeat the
        schedule; their noise is still keyed by the global index."""
        n = len(self.times) - 1
        return self.times[(t - 1) % n + 1]


def workload(name: str, **over) -> Workload:
    """The BASELINE.json configs as concrete seeded inputs."""
    if name == "C1":
        w = Workload("C1", 256, 256, 1, 8, None, 0, "c1")
    elif name == "C1plane":
        w = Workload("C1plane", 256, 256, 1, 8, None, 0, "plane")
    elif name == "C2":
        w = Workload("C2", 512, 512, 2, 11, 0.0, 1, "c2")
    elif name == "C3":
        w = Workload("C3", 1024, 1024, 100, 8, 10.0, 11, "diffusion",
                     [0.0] + [60.0 * k for k in range(1, 100)])
    elif name == "C4":
        w = Workload("C4", 2048, 2048, 200, 8, 10.0, 12, "diffusion",
                     [0.0] + [60.0 + 30.0 * k for k in range(1, 200)])
    elif name == "C5":
        w = Workload("C5", 2048, 2048, 2000, 8, 10.0, 13, "diffusion",
                     [0.0] + [60.0 + 3.0 * k for k in range(1, 2000)])
    else:
        raise ValueError(name)
    for k, v in over.items():
        setattr(w, k, v)
    if w.kind == "diffusion" and len(w.times) < w.T:
        raise ValueError("diffusion workload needs one time per frame")
    return w


def noise_generator(seed: int, t: int, device) -> torch.Generator:
    g = torch.Generator(device=device)
    g.manual_seed((int(seed) * 1_000_003 + int(t)) & 0x7FFF_FFFF_FFFF_FFFF)
    return g


def make_frame(w: Workload, t: int, device="cpu", snr_db="default") -> torch.Tensor:
    """Frame t of workload w as complex64 [H,W] on ``device``."""
    snr = w.snr_db if snr_db == "default" else snr_db
    ph = carrier_phase(w.H, w.W, device) + w.phase(t, device)
    g = torch.polar(torch.ones_like(ph), ph).to(torch.complex64)
    if snr is not None:
        sigma2 = 10.0 ** (-snr / 10.0)
        n = torch.randn(w.H, w.W, 2, generator=noise_generator(w.seed, t, device),
                        device=device, dtype=torch.float32)
        n = n * math.sqrt(sigma2 / 2.0)
        g = g + torch.view_as_complex(n)
    return g


def make_stack(w: Workload, frames=None, device="cpu", snr_db="default", out=None) -> torch.Tensor:
    """Frames ``frames`` (default all) of w as complex64 [T,H,W]; writes into ``out`` if given."""
    ts = list(range(w.T)) if frames is None else list(frames)
    if out is None:
        out = torch.empty(len(ts), w.H, w.W, dtype=torch.complex64, device=device)
    for j, t in enumerate(ts):
        out[j] = make_frame(w, t, device, snr_db)
    return out


def true_phase(w: Workload, t: int, device="cpu") -> torch.Tensor:
    """Analytic phase of frame t including the carrier (float64 [H,W], unwrapped)."""
    return carrier_phase(w.H, w.W, device) + w.phase(t, device)


def make_intensity_frame(w: Workload, t: int, device="cpu", snr_db="default", visibility: float = 0.45,
                         background: float = 0.5) -> torch.Tensor:
    """8-bit carrier fringe intensity of frame t (the camera-side input of row f1):
    I = 255·clip(b + v·cos(ω_c·r + φ_t) + n), n real Gaussian with E n² = v²/(2·10^{SNR/10}) (the
    SNR of the analytic signal the bandpass recovers, amplitude v/2), quantised to uint8."""
    snr = w.snr_db if snr_db == "default" else snr_db
    ph = carrier_phase(w.H, w.W, device) + w.phase(t, device)
    i = background + visibility * torch.cos(ph)
    if snr is not None:
        g = noise_generator(w.seed + 7919, t, device)
        sigma = visibility * math.sqrt(0.5 / (10.0 ** (snr / 10.0)))
        i = i + sigma * torch.randn(w.H, w.W, generator=g, device=device, dtype=torch.float64)
    return torch.clamp(torch.round(i * 255.0), 0, 255).to(torch.uint8)
