"""Device plumbing: torch owns device memory and streams; kernels are ours."""

import numpy as np

try:
    import torch
except ImportError:  # pragma: no cover
    torch = None


def require_cuda():
    if torch is None or not torch.cuda.is_available():
        raise RuntimeError("paper_1712_08565_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback for the MF-WQ hot path")


def stream_ptr():
    return torch.cuda.current_stream().cuda_stream


def is_device_tensor(v):
    return torch is not None and isinstance(v, torch.Tensor) and v.is_cuda


def is_pinned_host(v):
    return torch is not None and isinstance(v, torch.Tensor) and not v.is_cuda and v.is_pinned()


def to_device(v, n=None):
    """Return (contiguous fp64 CUDA tensor, came_from_host)."""
    require_cuda()
    if is_device_tensor(v):
        t = v.reshape(-1)
        if t.dtype != torch.float64:
            t = t.to(torch.float64)
        t = t.contiguous()
        host = False
    elif torch is not None and isinstance(v, torch.Tensor):  # host torch tensor (pinned -> async H2D)
        t = v.reshape(-1).to(dtype=torch.float64).to("cuda", non_blocking=v.is_pinned())
        host = "torch"
    else:
        a = np.ascontiguousarray(np.asarray(v, dtype=float).ravel())
        t = torch.from_numpy(a).to("cuda", non_blocking=False)
        host = True
    if n is not None and t.numel() != n:
        raise ValueError(f"expected vector of length {n}, got {t.numel()}")
    return t, host


def check_out(out, n):
    """Validate a caller-provided output buffer before its pointer reaches a kernel."""
    if not (is_device_tensor(out) and out.dtype == torch.float64 and out.is_contiguous()
            and out.numel() == int(n)):
        raise ValueError(f"out must be a contiguous float64 CUDA tensor of length {int(n)}")
    if out.device.index != torch.cuda.current_device():
        raise ValueError("out must live on the current CUDA device")
    return out


def empty(n):
    require_cuda()
    return torch.empty(int(n), dtype=torch.float64, device="cuda")


def zeros(n):
    require_cuda()
    return torch.zeros(int(n), dtype=torch.float64, device="cuda")


def back(t, host):
    if host == "torch":
        out = torch.empty(t.shape, dtype=t.dtype, pin_memory=True)
        out.copy_(t, non_blocking=True)
        torch.cuda.current_stream().synchronize()
        return out
    return t.cpu().numpy() if host else t
