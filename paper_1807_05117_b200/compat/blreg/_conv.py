"""numpy <-> device conversions at the compat boundary."""

import numpy as np
import torch


def dev(domain, x, complex_=None):
    """Host (or device) array -> tensor on the domain's device."""
    if isinstance(x, torch.Tensor):
        return x.to(domain.torch_device)
    a = np.asarray(x)
    if complex_ is None:
        complex_ = np.iscomplexobj(a)
    dt = np.complex128 if complex_ else np.float64
    return torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(domain.torch_device)


def host(t):
    """Tensor -> numpy (host copy); numpy and scalars pass through."""
    if isinstance(t, torch.Tensor):
        return t.detach().cpu().numpy()
    if isinstance(t, tuple):
        return tuple(host(x) for x in t)
    return t
