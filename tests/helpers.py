"""Shared test helpers: tolerance metric (SURVEY §8(c) protocol) and device/host conversions."""
import numpy as np


def rel_err(got, ref):
    """max_i |g_i - o_i| / max(|o_i|, rms(o)) — per-element relative error with an rms floor."""
    g = np.asarray(got, np.float64).reshape(-1)
    o = np.asarray(ref, np.float64).reshape(-1)
    if o.size == 0:
        return 0.0
    rms = float(np.sqrt(np.mean(o * o)))
    if rms == 0.0:
        return float(np.abs(g).max())
    return float((np.abs(g - o) / np.maximum(np.abs(o), rms)).max())


def to_dev(arrs):
    import torch
    return [torch.tensor(np.ascontiguousarray(a), device="cuda") for a in arrs]


def to_host(ts):
    return [t.detach().cpu().numpy() for t in ts]


def assert_state_parity(prog, old, gpu_new, ora_new, tol, what=""):
    """Carried state compared directly; parameters compared through their update (new - old),
    which isolates the gradient (the update is small next to the weight)."""
    for k, s in enumerate(prog.slots):
        g = np.asarray(gpu_new[k], np.float64)
        o = np.asarray(ora_new[k], np.float64)
        if s.param:
            # both sides store fp32: allow one fp32 ulp of the new value before comparing updates
            d_o = o - np.asarray(old[k], np.float64)
            slack = np.abs(np.spacing(np.asarray(ora_new[k], np.float32))).astype(np.float64)
            diff = np.maximum(np.abs(g - o) - slack, 0.0)
            d_g = d_o + np.sign(g - o) * diff
            touched = np.abs(d_o).reshape(d_o.shape[0], -1).max(axis=1) > 0 if d_o.ndim == 2 else None
            if touched is not None and not touched.all():
                # row-sparse update (embedding rows of the batch's words): each row is its own
                # segmented sum, so the rms floor is taken per touched row
                e = max([rel_err(d_g[r], d_o[r]) for r in np.nonzero(touched)[0]] +
                        [float(np.abs(d_g[~touched]).max()) if (~touched).any() else 0.0])
            else:
                e = rel_err(d_g, d_o)
        else:
            e = rel_err(g, o)
        assert e <= tol, f"{what} slot {s.name}: rel err {e:.3e} > {tol}"
