"""oracle.dpfamily — TEST INFRASTRUCTURE ONLY.  PARITY UNPINNED.

FP64 CPU restatement (torch autograd, float64) of the DeePMD-style operators
that the north star names but the reference does not implement (SURVEY.md
§8(a')): the smooth environment matrix, the per-neighbour-type
embedding net with the G^T.R.R^T.G descriptor contraction (DeePMD se_e2_a), and
a DPA2-style repformer layer stack with gated, smoothly switched neighbour
self-attention.  There is no reference function to pin these against; the
oracle follows the reference's own conventions instead — MlpT (tanh hidden
layers, linear output, weights row-major [out][in], inference.cpp:87-101), the
directed CSR NnInput with FP64 edge_dr = r_j - r_i (inference.hpp:18-38), energy
as a sum of per-atom energies, forces and virial from dE/d(edge_dr)
(inference.cpp:372-387) — and is validated by finite differences, rotation /
translation / permutation invariance and extensivity (tests/test_dpfamily.py).

Only tests/, __graft_entry__.smoke() and bench.py's CPU legs may import this.

Model definition (also DESIGN.md §11; the device kernels implement the same
function, hmdp_dp.cu):

  environment (edge e = i -> j, d = edge_dr, r = |d|):
    sw(r) = 1 (r < rcs);  u^3 (-6u^2 + 15u - 10) + 1, u = (r - rcs)/(rc - rcs)
            (rcs <= r < rc);  0 (r >= rc)                      [DeePMD smooth switch]
    s = sw / r;  R_e = (s, s d_x / r, s d_y / r, s d_z / r)  [smooth env matrix row]
  se_a descriptor (family "se_a"):
    G_e  = emb[t_j](s_e)                       MLP [1, 32, 32]
    A_i  = (1/nnorm) sum_e R_e^T G_e            [4, 32]
    D_i  = A_i[:, :axis]^T A_i                   [axis, 32] -> axis*32 features
    e_i  = fit(D_i) + ebias[t_i]                MLP [axis*32, 32, 1]
  repformer (family "repformer", depth = 1 + n_layers):
    g1_i = g1map(D_i)                            MLP [axis*32, 32, 32]
    g2_e = G_e;  h_e = R_e[1:4];  w_e = sw(r_e)
    per layer:
      q_e, k_e, v_e = Wq g2_e + bq, Wk g2_e + bk, Wv g2_e + bv
      l_ef  = ((q_e . k_f)/sqrt(32) + shift) w_e w_f - shift        (f in N(i))
      a_ef  = softmax_f(l_ef)
      b_ef  = a_ef w_e w_f (h_e . h_f)                  [gated, switched attention]
      g2_e <- g2_e + Wo (sum_f b_ef v_f) + bo
      P_j   = Wc g1_j + bc
      conv_i = (1/nnorm) sum_e w_e g2_e * P_j            (g2 after the attention)
      T_i    = (1/nnorm) sum_e h_e^T g2_e                [3, 32]
      grrg_i = T_i[:, :axis]^T T_i                        [axis, 32]
      g1_i <- g1_i + upd([conv_i, grrg_i])               MLP [32 + axis*32, 32, 32]
    e_i = fit(g1_i) + ebias[t_i]                         MLP [32, 32, 1]
  repflow (family "repflow", DPA3-style; depth = 1 + n_layers): as repformer, with
  the attention replaced by an edge/angle message over the angle neighbours
  A(i) = {e : r_e < rca} (omega_e = DeePMD switch between rcas and rca):
      c_ef   = u_e . u_f                              (cos of the angle j-i-k, f != e)
      z_ef   = tanh(wa c_ef + ba)                     elementwise, MLP [1, 32] "angle"
      v_f    = Wv g2_f + bv
      m_e    = (1/anorm) sum_{f in A(i), f != e} omega_e omega_f z_ef * v_f
      g2_e  <- g2_e + Wo m_e + bo
"""
from __future__ import annotations

import json
import math

import numpy as np

SHIFT = 20.0  # attention logit shift of the smooth softmax (DeePMD attnw_shift)


def _torch():
    import torch

    return torch


def _mlp(p, x):
    """MlpT::forward (inference.cpp:87-101): tanh on hidden layers, linear output."""
    torch = _torch()
    n = len(p["weights"])
    for layer in range(n):
        w = torch.tensor(p["weights"][layer], dtype=torch.float64).view(p["sizes"][layer + 1],
                                                                          p["sizes"][layer])
        b = torch.tensor(p["biases"][layer], dtype=torch.float64)
        x = x @ w.T + b
        if layer + 1 < n:
            x = torch.tanh(x)
    return x


def smooth_switch(r, rc, rcs):
    torch = _torch()
    u = ((r - rcs) / (rc - rcs)).clamp(0.0, 1.0)
    mid = u ** 3 * (-6.0 * u ** 2 + 15.0 * u - 10.0) + 1.0
    return torch.where(r < rcs, torch.ones_like(r), torch.where(r < rc, mid, torch.zeros_like(r)))


def _padded(n, offset, nbr):
    """CSR -> padded [n, m] neighbour table (row order = CSR order)."""
    cnt = np.diff(offset)
    m = max(int(cnt.max()) if n else 0, 1)
    idx = np.full((n, m), -1, dtype=np.int64)
    slot = np.full((n, m), -1, dtype=np.int64)
    for i in range(n):
        a, b = int(offset[i]), int(offset[i + 1])
        idx[i, : b - a] = nbr[a:b]
        slot[i, : b - a] = np.arange(a, b)
    return idx, slot


def energy_terms(model: dict, types, offset, nbr, dr_edges):
    """Per-atom energies from edge displacements dr_edges (torch [ne, 3] f64, may
    require grad).  Returns (e_atom [n], stages dict)."""
    torch = _torch()
    fam = model["family"]
    n = len(types)
    rc, rcs = float(model["rc_model"]), float(model["rc_smooth"])
    axis, nnorm = int(model["axis"]), float(model["nnorm"])
    idx_np, slot_np = _padded(n, np.asarray(offset), np.asarray(nbr))
    idx = torch.from_numpy(idx_np)
    slot = torch.from_numpy(slot_np)
    mask = (idx >= 0).to(torch.float64)  # [n, m]
    safe_slot = slot.clamp(min=0)
    far = torch.tensor([2.0 * rc, 0.0, 0.0], dtype=torch.float64)
    # (no edges at all: gather from a one-row stand-in, every slot is padding)
    src = dr_edges if dr_edges.shape[0] > 0 else far[None, :]
    d = torch.where((slot >= 0)[..., None], src[safe_slot], far)  # [n, m, 3]
    r = torch.sqrt((d * d).sum(-1))
    w = smooth_switch(r, rc, rcs) * mask
    s = w / r
    R = torch.cat([s[..., None], (s / r)[..., None] * d], dim=-1)  # [n, m, 4]
    t_nb = torch.from_numpy(np.asarray(types, dtype=np.int64))[idx.clamp(min=0)]
    G = torch.zeros(n, idx.shape[1], 32, dtype=torch.float64)
    for t, emb in enumerate(model["embeddings"]):
        sel = ((t_nb == t) & (idx >= 0)).to(torch.float64)[..., None]
        G = G + sel * _mlp(emb, s[..., None])
    A = torch.einsum("nmc,nmb->ncb", R, G) / nnorm  # [n, 4, 32]
    D = torch.einsum("nca,ncb->nab", A[:, :, :axis], A).reshape(n, axis * 32)
    stages = {"desc": D}
    ty = torch.from_numpy(np.asarray(types, dtype=np.int64))
    ebias = torch.tensor(model["energy_bias"], dtype=torch.float64)[ty]
    if fam == "se_a":
        return _mlp(model["fitting"], D)[:, 0] + ebias, stages
    if fam not in ("repformer", "repflow"):
        raise ValueError(f"dpfamily oracle: unknown family {fam}")
    g1 = _mlp(model["g1map"], D)
    g2 = G
    h = R[..., 1:4]
    ww = w[:, :, None] * w[:, None, :]  # [n, m, m]
    gate = torch.einsum("nec,nfc->nef", h, h)
    neg = torch.where(mask[:, None, :] > 0, torch.zeros_like(ww), torch.full_like(ww, -1e30))
    stages["g1"] = [g1]
    if fam == "repflow":
        # angle neighbours (r < rca) as a padded sub-list of each atom's edges
        rca, rcas = float(model["rc_angle"]), float(model["rc_angle_smooth"])
        anorm = float(model["anorm"])
        rn = r.detach().numpy()
        sel = [np.nonzero((slot_np[i] >= 0) & (rn[i] < rca))[0] for i in range(n)]
        ma = max(max((len(x) for x in sel), default=0), 1)
        aidx = np.zeros((n, ma), dtype=np.int64)
        amask_np = np.zeros((n, ma))
        for i, x in enumerate(sel):
            aidx[i, : len(x)] = x
            amask_np[i, : len(x)] = 1.0
        aidx_t = torch.from_numpy(aidx)
        amask = torch.from_numpy(amask_np)
        ra = torch.gather(r, 1, aidx_t)
        da = torch.gather(d, 1, aidx_t[..., None].expand(-1, -1, 3))
        om = smooth_switch(ra, rca, rcas) * amask
        ua = da / ra[..., None]
        cos = torch.einsum("nec,nfc->nef", ua, ua)
        pair = om[:, :, None] * om[:, None, :] * (1.0 - torch.eye(ma, dtype=torch.float64)) / anorm
    for layer in model["layers"]:
        if fam == "repformer":
            q = _mlp(layer["q"], g2)
            k = _mlp(layer["k"], g2)
            v = _mlp(layer["v"], g2)
            lg = torch.einsum("nec,nfc->nef", q, k) / math.sqrt(32.0)
            lg = (lg + SHIFT) * ww - SHIFT + neg
            a = torch.softmax(lg, dim=-1)
            b = a * ww * gate
            o = torch.einsum("nef,nfc->nec", b, v)
        else:
            v = _mlp(layer["v"], g2)
            va = torch.gather(v, 1, aidx_t[..., None].expand(-1, -1, 32))
            z = _mlp(layer["angle"], cos[..., None])  # [n, ma, ma, 32] (linear, then tanh)
            z = torch.tanh(z)
            oa = torch.einsum("nef,nefc,nfc->nec", pair, z, va)
            o = torch.zeros(n, idx.shape[1], 32, dtype=torch.float64)
            o = o.scatter_add(1, aidx_t[..., None].expand(-1, -1, 32), oa * amask[..., None])
        g2 = g2 + _mlp(layer["o"], o) * mask[..., None]
        P = _mlp(layer["c"], g1)  # [n, 32]
        Pn = P[idx.clamp(min=0)]
        conv = torch.einsum("nm,nmc->nc", w, g2 * Pn) / nnorm
        T = torch.einsum("nmc,nmb->ncb", h, g2) / nnorm
        grrg = torch.einsum("nca,ncb->nab", T[:, :, :axis], T).reshape(n, axis * 32)
        g1 = g1 + _mlp(layer["update"], torch.cat([conv, grrg], dim=-1))
        stages["g1"].append(g1)
    return _mlp(model["fitting"], g1)[:, 0] + ebias, stages


def evaluate(model, types, offset, nbr, dr, want_stages: bool = False):
    """Energy, per-atom energy, forces, virial9 (W_ab = -sum_e d_a g_b, g = dE/dd)
    and the scalar virial (trace), all atoms owned — the NnOutput contract
    (inference.hpp:40-44) for the DeePMD-style families."""
    torch = _torch()
    if isinstance(model, str):
        model = json.loads(model)
    n = len(types)
    offset = np.asarray(offset)
    nbr = np.asarray(nbr)
    dr_t = torch.tensor(np.asarray(dr, dtype=np.float64).reshape(-1, 3), requires_grad=True)
    e_atom, stages = energy_terms(model, types, offset, nbr, dr_t)
    E = e_atom.sum()
    if E.requires_grad:
        (g,) = torch.autograd.grad(E, dr_t)
        g = g.numpy()
    else:  # no edges: nothing depends on the geometry
        g = np.zeros((0, 3))
    src = np.repeat(np.arange(n), np.diff(offset))
    F = np.zeros((n, 3))
    np.add.at(F, src, g)
    np.add.at(F, nbr, -g)
    d = dr_t.detach().numpy()
    W9 = -(d[:, :, None] * g[:, None, :]).sum(0)
    out = {
        "energy": float(E.detach()),
        "per_atom": e_atom.detach().numpy(),
        "forces": F,
        "virial9": W9,
        "virial": float(np.trace(W9)),
        "edge_g": g,
    }
    if want_stages:
        out["desc"] = stages["desc"].detach().numpy()
        if "g1" in stages:
            out["g1"] = [x.detach().numpy() for x in stages["g1"]]
    return out


def energy_of_positions(model, types, pos, box, offset, nbr):
    """E(positions) on a FIXED neighbour list (minimum-image edge vectors), for
    finite-difference checks."""
    torch = _torch()
    if isinstance(model, str):
        model = json.loads(model)
    pos = np.asarray(pos, dtype=np.float64)
    src = np.repeat(np.arange(len(types)), np.diff(offset))
    d = pos[np.asarray(nbr)] - pos[src]
    L = np.asarray(box, dtype=np.float64)
    d = d - L * np.rint(d / L)
    with torch.no_grad():
        e, _ = energy_terms(model, types, offset, nbr, torch.from_numpy(d))
    return float(e.sum())
