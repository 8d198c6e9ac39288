"""Shared helpers for the parity tests."""
import numpy as np

import paper_2008_03324_b200 as F


def models_from_golden(g_models):
    quad = F.QuadraticVisibility(*g_models["quad_k"])
    gps = {}
    for ns in (30, 70):
        par = g_models[f"gp{ns}_par"]
        gps[ns] = F.GpVisibility(g_models[f"gp{ns}_zs"], F.SeKernelParams(par[2], par[3], par[4]), par[0], par[1],
                                 g_models[f"gp{ns}_kinv"])
    return {"quad": quad, "gp30": gps[30], "gp70": gps[70]}


def oracle_model(model):
    if isinstance(model, F.QuadraticVisibility):
        return ("quad", model.k2, model.k1, model.k0)
    return ("gp", model.samples, model.params.sigma2, model.params.length_scale)


def reference_order(field):
    """Field rows re-ordered to the reference's x-major linear order (dense fields)."""
    lin = field.config.linear_index(field.occupied_index3)
    return field.factors[np.argsort(lin)]


def trace_rel_l2(mine, ref):
    """Per-voxel relative L2 over the N_v trace vector."""
    return np.linalg.norm(mine - ref, axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-300)


def info_rel_fro(mine, ref):
    """Per-voxel max-entry |delta| / Frobenius norm of the reference row."""
    return np.abs(mine - ref).max(axis=1) / np.maximum(np.linalg.norm(ref, axis=1), 1e-300)


def oracle_field(oracle, model, centers, points, kind, sigma=1.0, mask=None):
    if isinstance(model, F.QuadraticVisibility):
        return oracle.build_quad_factors(centers, points, sigma, model.k2, model.k1, model.k0, kind == "trace", mask)
    return oracle.build_gp_factors(centers, points, sigma, model.samples, model.kinv, model.k_s, np.cos(model.alpha),
                                   kind == "trace", mask)
