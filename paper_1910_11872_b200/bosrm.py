"""Thin ctypes binding of libbosrm.so (C ABI: include/bos_rootmusic.h).

Argument marshalling only: every step of the demodulation runs in the library's sm_100a
kernels.  Functions carry the C names.  There is no fallback: if the library is missing,
or a tensor is not where the ABI says it must be, the call raises.
"""

from __future__ import annotations

import ctypes
import os

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
# BOS_LIBRARY overrides the library path (development A/B builds only)
LIB_PATH = os.environ.get("BOS_LIBRARY") or os.path.join(_PKG, "libbosrm.so")

BOS_OK = 0
BOS_ERR_INVALID_ARG = -1
BOS_ERR_UNSUPPORTED = -2
BOS_ERR_CUDA = -3

FLAG_NONCONVERGED = 1 << 0
FLAG_AMBIGUOUS = 1 << 1
FLAG_SMALL_GAP = 1 << 2
FLAG_LOW_AMPLITUDE = 1 << 3
FLAG_NONFINITE = 1 << 4
FLAG_BORDER = 1 << 5

WINDOW_LEN_MIN = 3
WINDOW_LEN_MAX = 32
MODEL_ORDER = 3

VARIANT_PAPER = 0   # Algorithm 1 as published
VARIANT_FB = 1      # row f4: forward–backward averaged covariances (not in the paper)
VARIANT_FP64 = 2    # row f4: the whole pixel in double precision (bit mask, combinable with FB)

# name -> (restype, argtypes); must match include/bos_rootmusic.h
_VP, _I, _SZ = ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t
SIGNATURES = {
    "bos_rootmusic_demod": (_I, [_VP, _I, _I, _I, _I, _I, _VP, _VP, _VP, _VP]),
    "bos_rootmusic_demod_stack": (_I, [_VP, _I, _I, _I, _I, _I, _I, _VP, _VP, _VP, _VP]),
    "bos_rootmusic_host_workspace_bytes": (_SZ, [_I, _I, _I, _I]),
    "bos_rootmusic_demod_stack_host": (_I, [_VP, _I, _I, _I, _I, _I, _I, _VP, _VP, _VP, _SZ, _I, _VP]),
    "bos_rootmusic_iteration_counts": (_I, [_VP, _I, _I, _I, _I, _I, _VP, _VP, _VP, _VP]),
    "bos_rootmusic_demod_ex": (_I, [_VP, _I, _I, _I, _I, _I, _VP, _VP, _VP, _VP, _VP, _VP]),
    "bos_rootmusic_demod_variant": (_I, [_VP, _I, _I, _I, _I, _I, _I, _I, _VP, _VP, _VP, _VP, _VP, _VP]),
    "bos_analytic_signal_workspace_bytes": (_SZ, [_I, _I, _I]),
    "bos_unwrap_workspace_bytes": (_SZ, [_I, _I, _I]),
    "bos_unwrap": (_I, [_VP, _I, _I, _I, _VP, _VP, _SZ, _VP]),
    "bos_analytic_signal": (_I, [_VP, _I, _I, _I, ctypes.c_double, ctypes.c_double, ctypes.c_double, _I, _VP, _VP,
                                 _SZ, _VP]),
    "bos_analytic_plan_create": (_I, [_I, _I, _I, ctypes.POINTER(ctypes.c_void_p), ctypes.POINTER(ctypes.c_size_t)]),
    "bos_analytic_signal_planned": (_I, [_VP, _VP, _I, ctypes.c_double, ctypes.c_double, ctypes.c_double, _I, _VP,
                                         _VP, _SZ, _VP]),
    "bos_analytic_plan_destroy": (_I, [_VP]),
    "bos_index_gradient": (_I, [_VP, _SZ, ctypes.c_double, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                _VP, _VP]),
    "bos_vertical_profile": (_I, [_VP, _I, _I, _I, _VP, _VP]),
    "bos_strerror": (ctypes.c_char_p, [_I]),
    "bos_abi_version": (_I, []),
}

_lib = None


class BosError(RuntimeError):
    def __init__(self, code: int, where: str):
        super().__init__(f"{where}: {bos_strerror(code)} (code {code})")
        self.code = code


def lib() -> ctypes.CDLL:
    """Load libbosrm.so (built in-tree by paper_1910_11872_b200.build); raise if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} is missing: build it with "
                               "`python -m paper_1910_11872_b200.build` (no CPU fallback exists)")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            if "BOS_LIBRARY" in os.environ and not hasattr(L, name):
                continue                      # A/B builds of older revisions may lack new entries
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def bos_strerror(code: int) -> str:
    return lib().bos_strerror(int(code)).decode()


def bos_abi_version() -> int:
    return lib().bos_abi_version()


def _check(rc: int, where: str):
    if rc != BOS_OK:
        raise BosError(rc, where)


def _stream_for(stream, device: torch.device) -> torch.cuda.Stream:
    """The stream a call runs on: ``stream`` (must belong to ``device``) or the device's current
    stream (not the current device's: the tensors decide where the work runs)."""
    if stream is None:
        return torch.cuda.current_stream(device)
    if stream.device != device:
        raise ValueError(f"stream is on {stream.device}, the tensors on {device}")
    return stream


def _keep_alive(stream: torch.cuda.Stream, device: torch.device, *tensors):
    """Tensors allocated here (on the current stream) but used by work queued on another
    stream: tell the caching allocator, so the memory is not reused before that work ends."""
    if stream != torch.cuda.current_stream(device):
        for t in tensors:
            if t is not None:
                t.record_stream(stream)


def _dev_tensor(t: torch.Tensor, dtype, name: str, device: torch.device | None = None,
                numel: int | None = None) -> torch.Tensor:
    """A caller-supplied CUDA tensor the C ABI reads or writes through a bare pointer: the
    library cannot see sizes, so dtype, contiguity, device and element count are checked here."""
    if not isinstance(t, torch.Tensor) or t.device.type != "cuda":
        raise ValueError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise ValueError(f"{name} must be {dtype}, got {t.dtype}")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    if device is not None and t.device != device:
        raise ValueError(f"{name} is on {t.device}, frames on {device}")
    if numel is not None and t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, the call needs {numel}")
    return t


def _host_tensor(t: torch.Tensor, dtype, name: str, numel: int) -> torch.Tensor:
    if not isinstance(t, torch.Tensor) or t.device.type != "cpu" or t.dtype != dtype or not t.is_contiguous():
        raise ValueError(f"{name} must be a contiguous CPU {dtype} tensor")
    if t.numel() != numel:
        raise ValueError(f"{name} has {t.numel()} elements, the call needs {numel}")
    return t


def _frames3(frames: torch.Tensor) -> torch.Tensor:
    if frames.dim() == 2:
        frames = frames.unsqueeze(0)
    if frames.dim() != 3:
        raise ValueError("frames must be [H,W] or [T,H,W]")
    return frames


def _opt_flags(flags, T, H, W, device):
    """flags=True → allocate [T,H,W] uint8; a tensor → checked, written in place; None/False → skip."""
    if flags is True:
        return torch.empty(T, H, W, dtype=torch.uint8, device=device)
    if flags is None or flags is False:
        return None
    return _dev_tensor(flags, torch.uint8, "flags", device, T * H * W)


def _ptr(t):
    return t.data_ptr() if t is not None else None


def bos_rootmusic_demod(frames: torch.Tensor, window_len: int = 8, model_order: int = MODEL_ORDER,
                        ref_phase: torch.Tensor | None = None, out_phase: torch.Tensor | None = None,
                        flags: torch.Tensor | bool | None = None, stream=None):
    """Demodulate complex64 CUDA frames [T,H,W] (or [H,W]) → (phase float32, flags uint8|None).

    ``flags=True`` allocates the flag plane; a tensor is written in place; None skips it."""
    frames = _dev_tensor(_frames3(frames), torch.complex64, "frames")
    T, H, W = frames.shape
    dev = frames.device
    s = _stream_for(stream, dev)
    if out_phase is None:
        out_phase = torch.empty(T, H, W, dtype=torch.float32, device=dev)
    _dev_tensor(out_phase, torch.float32, "out_phase", dev, T * H * W)
    flags = _opt_flags(flags, T, H, W, dev)
    if ref_phase is not None:
        _dev_tensor(ref_phase, torch.float32, "ref_phase", dev, H * W)
    _keep_alive(s, dev, out_phase, flags)
    with torch.cuda.device(dev):
        rc = lib().bos_rootmusic_demod(frames.data_ptr(), T, H, W, int(window_len), int(model_order),
                                       _ptr(ref_phase), out_phase.data_ptr(), _ptr(flags), s.cuda_stream)
    _check(rc, "bos_rootmusic_demod")
    return out_phase, flags


def bos_rootmusic_demod_stack(frames: torch.Tensor, window_len: int = 8, model_order: int = MODEL_ORDER,
                              ref_index: int = 0, ref_phase_out: torch.Tensor | None = None,
                              out_phase: torch.Tensor | None = None, flags=None, stream=None):
    """Time-lapse stack against frames[ref_index] → (phase, flags|None, ref_phase)."""
    frames = _dev_tensor(_frames3(frames), torch.complex64, "frames")
    T, H, W = frames.shape
    dev = frames.device
    s = _stream_for(stream, dev)
    if ref_phase_out is None:
        ref_phase_out = torch.empty(H, W, dtype=torch.float32, device=dev)
    if out_phase is None:
        out_phase = torch.empty(T, H, W, dtype=torch.float32, device=dev)
    flags = _opt_flags(flags, T, H, W, dev)
    _dev_tensor(ref_phase_out, torch.float32, "ref_phase_out", dev, H * W)
    _dev_tensor(out_phase, torch.float32, "out_phase", dev, T * H * W)
    _keep_alive(s, dev, ref_phase_out, out_phase, flags)
    with torch.cuda.device(dev):
        rc = lib().bos_rootmusic_demod_stack(frames.data_ptr(), T, H, W, int(window_len), int(model_order),
                                             int(ref_index), ref_phase_out.data_ptr(), out_phase.data_ptr(),
                                             _ptr(flags), s.cuda_stream)
    _check(rc, "bos_rootmusic_demod_stack")
    return out_phase, flags, ref_phase_out


def bos_rootmusic_host_workspace_bytes(H: int, W: int, chunk_frames: int, with_flags: bool) -> int:
    return int(lib().bos_rootmusic_host_workspace_bytes(int(H), int(W), int(chunk_frames), int(bool(with_flags))))


def bos_rootmusic_demod_stack_host(h_frames: torch.Tensor, window_len: int = 8, model_order: int = MODEL_ORDER,
                                   ref_index: int = 0, h_out_phase: torch.Tensor | None = None,
                                   h_flags=None, workspace: torch.Tensor | None = None, chunk_frames: int = 8,
                                   stream=None, device=None):
    """Host-buffer stack demod: CPU complex64 [T,H,W] (pinned for overlap) → CPU phase/flags.
    The device workspace is a caller-owned CUDA uint8 tensor (allocated here if None; it
    decides the device, else ``device``, else the current device).  The call is asynchronous:
    results are valid after ``stream`` (default: the device's current stream) synchronises."""
    h_frames = _frames3(h_frames)
    if h_frames.device.type != "cpu" or h_frames.dtype != torch.complex64 or not h_frames.is_contiguous():
        raise ValueError("h_frames must be a contiguous CPU complex64 tensor")
    T, H, W = h_frames.shape
    pin = h_frames.is_pinned()
    if h_out_phase is None:
        h_out_phase = torch.empty(T, H, W, dtype=torch.float32, pin_memory=pin)
    _host_tensor(h_out_phase, torch.float32, "h_out_phase", T * H * W)
    if h_flags is True:
        h_flags = torch.empty(T, H, W, dtype=torch.uint8, pin_memory=pin)
    elif h_flags is False:
        h_flags = None
    if h_flags is not None:
        _host_tensor(h_flags, torch.uint8, "h_flags", T * H * W)
    need = bos_rootmusic_host_workspace_bytes(H, W, min(chunk_frames, T), h_flags is not None)
    if workspace is None:
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    dev = workspace.device
    _dev_tensor(workspace, torch.uint8, "workspace")
    if workspace.numel() < need:
        raise ValueError(f"workspace has {workspace.numel()} bytes, the call needs {need}")
    s = _stream_for(stream, dev)
    _keep_alive(s, dev, workspace)
    with torch.cuda.device(dev):
        rc = lib().bos_rootmusic_demod_stack_host(
            h_frames.data_ptr(), T, H, W, int(window_len), int(model_order), int(ref_index),
            h_out_phase.data_ptr(), _ptr(h_flags), workspace.data_ptr(), workspace.numel(), int(chunk_frames),
            s.cuda_stream)
    _check(rc, "bos_rootmusic_demod_stack_host")
    return h_out_phase, h_flags


def bos_rootmusic_iteration_counts(frames: torch.Tensor, window_len: int = 8, model_order: int = MODEL_ORDER,
                                   ref_phase: torch.Tensor | None = None, stream=None):
    """Run the counting variant; returns dict(pixels, power_its, aberth_y, aberth_x) (host ints)."""
    frames = _dev_tensor(_frames3(frames), torch.complex64, "frames")
    T, H, W = frames.shape
    dev = frames.device
    s = _stream_for(stream, dev)
    out = torch.empty(T, H, W, dtype=torch.float32, device=dev)
    cnt = torch.zeros(4, dtype=torch.int64, device=dev)
    if ref_phase is not None:
        _dev_tensor(ref_phase, torch.float32, "ref_phase", dev, H * W)
    _keep_alive(s, dev, out, cnt)
    with torch.cuda.device(dev):
        rc = lib().bos_rootmusic_iteration_counts(frames.data_ptr(), T, H, W, int(window_len), int(model_order),
                                                  _ptr(ref_phase), out.data_ptr(), cnt.data_ptr(), s.cuda_stream)
    _check(rc, "bos_rootmusic_iteration_counts")
    s.synchronize()
    c = cnt.cpu().tolist()
    return dict(pixels=c[0], power_its=c[1], aberth_y=c[2], aberth_x=c[3], out=out)


def bos_rootmusic_demod_ex(frames: torch.Tensor, window_len: int = 8, model_order: int = MODEL_ORDER,
                           ref_phase: torch.Tensor | None = None, flags=None, omega=True, stream=None):
    """bos_rootmusic_demod plus the Eq.(15) local frequency maps → (phase, flags|None, ω_x, ω_y)."""
    return bos_rootmusic_demod_variant(frames, window_len, model_order, VARIANT_PAPER, ref_phase, None, flags,
                                       omega, stream, 0, _entry="bos_rootmusic_demod_ex")


def bos_rootmusic_demod_variant(frames: torch.Tensor, window_len: int = 8, model_order: int = MODEL_ORDER,
                                variant: int = VARIANT_FB, ref_phase: torch.Tensor | None = None,
                                out_phase: torch.Tensor | None = None, flags=None, omega=False, stream=None,
                                subarray_len: int = 0, _entry: str = "bos_rootmusic_demod_variant"):
    """bos_rootmusic_demod_ex with the row-f4 variants: ``variant`` a mask of VARIANT_FB /
    VARIANT_FP64, ``subarray_len`` m < window_len for spatial smoothing (0 = none)
    → (phase, flags|None, ω_x|None, ω_y|None)."""
    frames = _dev_tensor(_frames3(frames), torch.complex64, "frames")
    T, H, W = frames.shape
    dev = frames.device
    s = _stream_for(stream, dev)
    out = out_phase if out_phase is not None else torch.empty(T, H, W, dtype=torch.float32, device=dev)
    _dev_tensor(out, torch.float32, "out_phase", dev, T * H * W)
    fl = _opt_flags(flags, T, H, W, dev)
    wx = torch.empty(T, H, W, dtype=torch.float32, device=dev) if omega else None
    wy = torch.empty(T, H, W, dtype=torch.float32, device=dev) if omega else None
    if ref_phase is not None:
        _dev_tensor(ref_phase, torch.float32, "ref_phase", dev, H * W)
    _keep_alive(s, dev, out, fl, wx, wy)
    with torch.cuda.device(dev):
        if _entry == "bos_rootmusic_demod_ex":
            rc = lib().bos_rootmusic_demod_ex(frames.data_ptr(), T, H, W, int(window_len), int(model_order),
                                              _ptr(ref_phase), out.data_ptr(), _ptr(fl), _ptr(wx), _ptr(wy),
                                              s.cuda_stream)
        else:
            rc = lib().bos_rootmusic_demod_variant(
                frames.data_ptr(), T, H, W, int(window_len), int(subarray_len), int(model_order), int(variant),
                _ptr(ref_phase), out.data_ptr(), _ptr(fl), _ptr(wx), _ptr(wy), s.cuda_stream)
    _check(rc, _entry)
    return out, fl, wx, wy


def bos_index_gradient(phase: torch.Tensor, n0: float, mu: float, f_x: float, cell_len: float,
                       out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Eq.(17): ∂n/∂x = n0 / (2 μ f_x L²) · φ on a CUDA float32 tensor (any shape)."""
    _dev_tensor(phase, torch.float32, "phase")
    dev = phase.device
    s = _stream_for(stream, dev)
    if out is None:
        out = torch.empty_like(phase)
    _dev_tensor(out, torch.float32, "out", dev, phase.numel())
    _keep_alive(s, dev, out)
    with torch.cuda.device(dev):
        rc = lib().bos_index_gradient(phase.data_ptr(), phase.numel(), float(n0), float(mu), float(f_x),
                                      float(cell_len), out.data_ptr(), s.cuda_stream)
    _check(rc, "bos_index_gradient")
    return out


def bos_vertical_profile(phase: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Row f3: column-averaged phase per row of a CUDA float32 [T,H,W] (or [H,W]) → [T,H] (or [H])."""
    squeeze = phase.dim() == 2
    ph = _dev_tensor(phase.unsqueeze(0) if squeeze else phase, torch.float32, "phase")
    if ph.dim() != 3:
        raise ValueError("phase must be [H,W] or [T,H,W]")
    T, H, W = ph.shape
    dev = ph.device
    s = _stream_for(stream, dev)
    if out is None:
        out = torch.empty(T, H, dtype=torch.float32, device=dev)
    _dev_tensor(out, torch.float32, "out", dev, T * H)
    _keep_alive(s, dev, out)
    with torch.cuda.device(dev):
        rc = lib().bos_vertical_profile(ph.data_ptr(), T, H, W, out.data_ptr(), s.cuda_stream)
    _check(rc, "bos_vertical_profile")
    return out[0] if squeeze and out.dim() == 2 and out.shape[0] == 1 else out


def bos_analytic_signal(frames_u8: torch.Tensor, fx: float, fy: float, radius: float, remove_carrier: bool = False,
                        out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
                        stream=None) -> torch.Tensor:
    """Row f1: uint8 CUDA frames [T,H,W] (or [H,W]) → analytic signal Γ complex64 [T,H,W]."""
    frames_u8 = _dev_tensor(_frames3(frames_u8), torch.uint8, "frames_u8")
    T, H, W = frames_u8.shape
    dev = frames_u8.device
    s = _stream_for(stream, dev)
    if out is None:
        out = torch.empty(T, H, W, dtype=torch.complex64, device=dev)
    _dev_tensor(out, torch.complex64, "out", dev, T * H * W)
    need = int(lib().bos_analytic_signal_workspace_bytes(H, W, T))
    if workspace is None:
        workspace = torch.empty(max(need, 256), dtype=torch.uint8, device=dev)
    _dev_tensor(workspace, torch.uint8, "workspace", dev)
    _keep_alive(s, dev, out, workspace)
    with torch.cuda.device(dev):
        rc = lib().bos_analytic_signal(frames_u8.data_ptr(), T, H, W, float(fx), float(fy), float(radius),
                                       int(bool(remove_carrier)), out.data_ptr(), workspace.data_ptr(),
                                       workspace.numel(), s.cuda_stream)
    _check(rc, "bos_analytic_signal")
    return out


class AnalyticPlan:
    """Caller-owned cuFFT plans for row f1 (bos_analytic_plan_create / _destroy): repeated
    bos_analytic_signal_planned calls on H×W frames make no plans and do not synchronise.
    close() (and garbage collection) waits for the last planned call before destroying the
    plans and releasing the work area (bos_rootmusic.h: no planned call may still run)."""

    def __init__(self, H: int, W: int, max_frames: int, device=None):
        dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        if dev.index is None:
            dev = torch.device("cuda", torch.cuda.current_device())
        self.device = dev
        self._h = ctypes.c_void_p()
        ws = ctypes.c_size_t()
        with torch.cuda.device(dev):
            _check(lib().bos_analytic_plan_create(int(H), int(W), int(max_frames), ctypes.byref(self._h),
                                                  ctypes.byref(ws)), "bos_analytic_plan_create")
        self.H, self.W, self.max_frames = int(H), int(W), int(max_frames)
        self.workspace = torch.empty(max(int(ws.value), 256), dtype=torch.uint8, device=dev)
        self._last = None          # event recorded after the last planned call

    def _record(self, stream: torch.cuda.Stream):
        ev = torch.cuda.Event()
        ev.record(stream)
        self._last = ev

    def close(self):
        if self._h is not None and self._h.value:
            if self._last is not None:
                self._last.synchronize()      # no planned call may still run (header contract)
            with torch.cuda.device(self.device):
                lib().bos_analytic_plan_destroy(self._h)
        self._h = None
        self._last = None
        self.workspace = None

    def __del__(self):
        try:
            self.close()
        except Exception:       # interpreter shutdown
            pass


def bos_analytic_signal_planned(plan: AnalyticPlan, frames_u8: torch.Tensor, fx: float, fy: float, radius: float,
                                remove_carrier: bool = False, out: torch.Tensor | None = None,
                                stream=None) -> torch.Tensor:
    """Row f1 with a plan (AnalyticPlan): uint8 CUDA [T,H,W] → Γ complex64 [T,H,W], asynchronous."""
    if plan._h is None:
        raise ValueError("the plan is closed")
    frames_u8 = _dev_tensor(_frames3(frames_u8), torch.uint8, "frames_u8", plan.device)
    T, H, W = frames_u8.shape
    if (H, W) != (plan.H, plan.W):
        raise ValueError(f"plan is for {plan.H}x{plan.W} frames, got {H}x{W}")
    dev = plan.device
    s = _stream_for(stream, dev)
    if out is None:
        out = torch.empty(T, H, W, dtype=torch.complex64, device=dev)
    _dev_tensor(out, torch.complex64, "out", dev, T * H * W)
    _keep_alive(s, dev, out, plan.workspace)
    with torch.cuda.device(dev):
        rc = lib().bos_analytic_signal_planned(plan._h, frames_u8.data_ptr(), T, float(fx), float(fy), float(radius),
                                               int(bool(remove_carrier)), out.data_ptr(), plan.workspace.data_ptr(),
                                               plan.workspace.numel(), s.cuda_stream)
    _check(rc, "bos_analytic_signal_planned")
    plan._record(s)
    return out


def bos_unwrap(wrapped: torch.Tensor, out: torch.Tensor | None = None, workspace: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
    """Row f2: Herráez reliability-sorted unwrapping of CUDA float32 [T,H,W] (or [H,W]) phase maps."""
    w = _dev_tensor(_frames3(wrapped), torch.float32, "wrapped")
    T, H, W = w.shape
    dev = w.device
    s = _stream_for(stream, dev)
    if out is None:
        out = torch.empty_like(w)
    _dev_tensor(out, torch.float32, "out", dev, T * H * W)
    need = int(lib().bos_unwrap_workspace_bytes(H, W, T)) or int(lib().bos_unwrap_workspace_bytes(H, W, 1))
    if workspace is None:
        workspace = torch.empty(need, dtype=torch.uint8, device=dev)
    _dev_tensor(workspace, torch.uint8, "workspace", dev)
    _keep_alive(s, dev, out, workspace)
    with torch.cuda.device(dev):
        rc = lib().bos_unwrap(w.data_ptr(), T, H, W, out.data_ptr(), workspace.data_ptr(), workspace.numel(),
                              s.cuda_stream)
    _check(rc, "bos_unwrap")
    return out.view(wrapped.shape)
