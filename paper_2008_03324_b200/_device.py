"""Device plumbing: torch for allocation, streams and H2D/D2H copies."""
from __future__ import annotations

import numpy as np
import torch


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2008_03324_b200 compute requires a CUDA device (B200); none is visible")
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise ValueError(f"device must be a CUDA device, got {d}")
    return d


def stream_handle(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def to_device_f64(x, device: torch.device, shape_tail=None) -> torch.Tensor:
    """float64 C-contiguous device tensor from numpy / torch input (float32 promoted exactly)."""
    if isinstance(x, torch.Tensor):
        t = x.to(device=device, dtype=torch.float64)
    else:
        a = np.asarray(x, dtype=np.float64)
        t = torch.from_numpy(np.ascontiguousarray(a)).to(device=device, non_blocking=False)
    if shape_tail is not None:
        t = t.reshape(-1, *shape_tail)
    return t.contiguous()


def to_numpy(t: torch.Tensor) -> np.ndarray:
    return t.detach().cpu().numpy()
