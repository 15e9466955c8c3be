"""Float64 NumPy implementation of the per-rank domain-decomposition phases
(TEST INFRASTRUCTURE).  It follows the same phase program as the CUDA engine
(paper_2602_02234_b200.dd.GpuEngine / hmdp_dd_phase) so the DD host logic --
plans, halo maps, transports, phase ordering -- can be checked on CPU, with
gloo, against the single-domain oracle.  Math follows the reference network
(/root/reference/proj/src/nn/inference.cpp:183-416) in the algebraically
regrouped form used by the kernels (message-MLP linearity)."""
from __future__ import annotations

import json

import numpy as np
import torch


def _mlp(m):
    W1 = np.array(m["weights"][0]).reshape(m["sizes"][1], m["sizes"][0])
    W2 = np.array(m["weights"][1]).reshape(m["sizes"][2], m["sizes"][1])
    return W1, np.array(m["biases"][0]), W2, np.array(m["biases"][1])


class NumpyEngine:
    def __init__(self, model: dict | str):
        if isinstance(model, str):
            model = json.loads(model)
        self.m = model
        self.rc = float(model["rc_model"])
        self.mu = np.array(model["basis"]["centers"])
        self.width = float(model["basis"]["width"])
        self.K = self.mu.shape[0]
        self.H = int(model["hidden"])
        self.nt = int(model["n_types"])
        self.embed = _mlp(model["embedding"])
        self.fit = _mlp(model["fitting"])
        self.msg = [_mlp(l["message"]) for l in model["layers"]]
        self.upd = [_mlp(l["update"]) for l in model["layers"]]
        self.M = len(self.msg)

    # ---- rows exchanged by the driver (torch CPU views of numpy storage) ----
    def p_rows(self):
        return self.t_p

    def remote_rows(self):
        return self.t_rem

    def ghost_sum_rows(self):
        return self.t_gs

    def force_rows(self):
        return self.t_f

    def index(self, idx):
        return torch.as_tensor(np.asarray(idx, dtype=np.int64))

    def setup(self, plan):
        self.n = plan.n_loc
        self.no = plan.n_own
        off = np.asarray(plan.offset)
        self.src = np.repeat(np.arange(self.n), np.diff(off))
        self.tgt = np.asarray(plan.nbr, dtype=np.int64)
        self.ty = np.asarray(plan.types)
        dr = np.asarray(plan.dr).reshape(-1, 3)
        r = np.linalg.norm(dr, axis=1)
        self.r, self.u, self.dr = r, dr / r[:, None], dr
        on = 0.9 * self.rc
        x = np.pi * (r - on) / (0.1 * self.rc)
        mid = (r > on) & (r < self.rc)
        self.s = np.where(r <= on, 1.0, np.where(r >= self.rc, 0.0, 0.5 * (np.cos(x) + 1.0)))
        self.ds = np.where(mid, -0.5 * np.sin(x) * np.pi / (0.1 * self.rc), 0.0)
        d = r[:, None] - self.mu[None, :]
        gk = np.exp(-d * d / (2 * self.width ** 2))
        self.b = gk * self.s[:, None]
        self.db = -d / self.width ** 2 * gk * self.s[:, None] + gk * self.ds[:, None]
        self.p = np.zeros((self.n, self.H))
        self.rem = np.zeros((self.n, self.H))
        self.gs = np.zeros((self.n, self.H))
        self.f = np.zeros((self.n, 3))
        self.t_p, self.t_rem = torch.from_numpy(self.p), torch.from_numpy(self.rem)
        self.t_gs, self.t_f = torch.from_numpy(self.gs), torch.from_numpy(self.f)
        self.g = np.zeros(self.src.shape[0])
        self.e_atom = np.zeros(self.n)
        self.h = [np.zeros((self.n, self.H)) for _ in range(self.M + 1)]
        self.z = [None] * max(self.M, 1)
        self.D = [None, None]
        self.pe = [None, None]
        self.uz = [None] * max(self.M, 1)
        self.own = np.zeros((self.n, self.H))

    def _fit(self, hM):
        W1, b1, W2, b2 = self.fit
        z = np.tanh(hM @ W1.T + b1)
        e = z @ W2[0] + b2[0]
        dz = W2[0][None, :] * (1.0 - z * z)
        return e, dz @ W1

    def _gather(self, D):
        S = np.zeros((self.n, self.H))
        np.add.at(S, self.tgt, D)
        return S

    def _msg_backward(self, l, dh, first):
        W1u, b1u, W2u, b2u = self.upd[l]
        W1m, b1m, W2m, b2m = self.msg[l]
        H = self.H
        zu = self.uz[l]
        dz = (dh @ W2u) * (1.0 - zu * zu)
        din = dz @ W1u
        o = slice(0, self.no)
        self.own[o] = dh[o] + din[o, :H]
        dmsum = din[:, H:]
        v = dmsum @ W2m        # v[i, k] = sum_c W2[c][k] dmsum[i][c]
        c0 = dmsum @ b2m
        vs = v[self.src]
        z = self.z[l]
        d = self.s[:, None] * vs * (1.0 - z * z)
        wv = self.db @ W1m[:, H:].T
        tot = np.sum(self.ds[:, None] * vs * z + d * wv, axis=1) + self.ds * c0[self.src]
        self.g = tot if first else self.g + tot
        self.D[l & 1] = d

    def phase(self, ph, l=0):
        H, K, no = self.H, self.K, self.no
        if ph == 0:
            desc = np.zeros((self.n, self.nt * K))
            for t in range(self.nt):
                sel = self.ty[self.tgt] == t
                np.add.at(desc[:, t * K:(t + 1) * K], self.src[sel], self.b[sel])
            W1, b1, W2, b2 = self.embed
            self.ez = np.tanh(desc @ W1.T + b1)
            h0 = self.ez @ W2.T + b2
            self.h[0][:no] = h0[:no]
            if self.M == 0:
                e, dh = self._fit(h0)
                self.e_atom[:no] = e[:no]
                dz1 = (dh @ W2) * (1.0 - self.ez ** 2)
                dd = dz1 @ W1
                self.g = np.sum(dd[self.src].reshape(-1, self.nt, K)[np.arange(self.src.shape[0]), self.ty[self.tgt]] * self.db, axis=1)
            else:
                self.p[:no] = (h0 @ self.msg[0][0][:, :H].T)[:no]
        elif ph == 1:
            self.pe[l & 1] = self.p[self.tgt].copy()
        elif ph == 2:
            W1m, b1m, W2m, b2m = self.msg[l]
            W1u, b1u, W2u, b2u = self.upd[l]
            z = np.tanh(self.pe[l & 1] + b1m + self.b @ W1m[:, H:].T)
            self.z[l] = z
            acc = np.zeros((self.n, H))
            np.add.at(acc, self.src, self.s[:, None] * z)
            ss = np.zeros(self.n)
            np.add.at(ss, self.src, self.s)
            msum = acc @ W2m.T + ss[:, None] * b2m
            hi = self.h[l]
            zu = np.tanh(np.concatenate([hi, msum], axis=1) @ W1u.T + b1u)
            self.uz[l] = zu
            hn = hi + zu @ W2u.T + b2u
            self.h[l + 1][:no] = hn[:no]
            if l < self.M - 1:
                self.p[:no] = (hn @ self.msg[l + 1][0][:, :H].T)[:no]
            else:
                e, dh = self._fit(hn)
                self.e_atom[:no] = e[:no]
                self._msg_backward(l, dh, True)
        elif ph == 3:
            S = self._gather(self.D[l & 1])
            self.gs[no:] = S[no:]
        elif ph == 4:
            S = self._gather(self.D[(l + 1) & 1]) + self.rem
            dh = self.own + S @ self.msg[l + 1][0][:, :H]
            self._msg_backward(l, dh, False)
        elif ph == 5:
            S = self._gather(self.D[0]) + self.rem
            dh = self.own + S @ self.msg[0][0][:, :H]
            W1, b1, W2, b2 = self.embed
            dz1 = (dh @ W2) * (1.0 - self.ez ** 2)
            dd = dz1 @ W1
            self.g = self.g + np.sum(dd[self.src].reshape(-1, self.nt, K)[np.arange(self.src.shape[0]), self.ty[self.tgt]] * self.db, axis=1)
        elif ph == 6:
            fe = self.u * self.g[:, None]
            self.f[:] = 0.0
            np.add.at(self.f, self.src, fe)
            np.add.at(self.f, self.tgt, -fe)
            self.W = -np.sum(self.g * self.r)
            self.W9 = -np.einsum("e,ea,eb->ab", self.g, self.dr, self.u).reshape(9)

    def result(self):
        return float(np.sum(self.e_atom[: self.no])), float(self.W), self.W9
