"""TEST INFRASTRUCTURE ONLY — numpy fp64 restatement of the placement policy.

Restates /root/reference/pkg/src/devplace/policy.py for use as the CPU parity
checker and CPU baseline; the product path never imports it.

* parameter layout / init      policy.py:41-42, 120-188
* group features               policy.py:97-114 (vocab: policy.py:57-66)
* input assembly               policy.py:256-263
* LSTM cell (gate order i,f,o,g) policy.py:220-233
* encoder / attention decoder  policy.py:271-314
* sampling rule                policy.py:317-326
* teacher-forced log-prob      policy.py:329-340
* analytic gradient            policy.py:236-253, 351-409

Per-step arithmetic uses the same numpy expressions (matvec over the
concatenated [x; h], separate elementwise products) so results agree with the
reference to the last bit on the same numpy build; tests pin that against
tests/golden/policy_*.npz.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

FIELD_ORDER = ("type_table", "dev_table", "w_enc", "b_enc", "w_dec", "b_dec", "w_att", "w_out", "b_out")


@dataclass(frozen=True)
class Dims:
    vocab_rows: int  # len(vocab) + 1 (last row: unknown types)
    n_dev: int
    hidden: int = 64
    dev_dim: int = 16
    type_dim: int = 16
    shape_slots: int = 8
    adj_slots: int = 64

    @property
    def feat(self) -> int:
        return self.type_dim + self.shape_slots + self.adj_slots

    def shapes(self):
        F, H, dd, D = self.feat, self.hidden, self.dev_dim, self.n_dev
        return {
            "type_table": (self.vocab_rows, self.type_dim), "dev_table": (D + 1, dd),
            "w_enc": (F + H, 4 * H), "b_enc": (4 * H,), "w_dec": (dd + H, 4 * H),
            "b_dec": (4 * H,), "w_att": (H, H), "w_out": (2 * H, dd), "b_out": (D,),
        }

    @property
    def n_params(self) -> int:
        return sum(int(np.prod(s)) for s in self.shapes().values())


def split_flat(flat, dims: Dims) -> dict:
    out, pos = {}, 0
    for name in FIELD_ORDER:
        shp = dims.shapes()[name]
        cnt = int(np.prod(shp))
        out[name] = np.asarray(flat[pos:pos + cnt], np.float64).reshape(shp)
        pos += cnt
    return out


def join_flat(arrs: dict) -> np.ndarray:
    return np.concatenate([np.ravel(arrs[k]) for k in FIELD_ORDER])


def init_flat(dims: Dims, seed: int = 0, scale: float = 0.1) -> np.ndarray:
    """Uniform[-scale, scale] per field in canonical order (policy.py:154-162)."""
    gen = np.random.default_rng(seed)
    return np.concatenate([gen.uniform(-scale, scale, size=s).ravel()
                           for s in (dims.shapes()[k] for k in FIELD_ORDER)])


def vocab_of(gg) -> list[str]:
    return sorted({op.op_type for op in gg.graph.ops})


@dataclass
class Features:
    order: list
    type_idx: list
    shape: np.ndarray
    adj: np.ndarray


def features(gg, vocab, shape_slots=8, adj_slots=64) -> Features:
    unknown = len(vocab)
    lookup = {t: i for i, t in enumerate(vocab)}
    order = list(gg.topo)
    T = len(order)
    shape = np.zeros((T, shape_slots))
    adj = np.zeros((T, adj_slots))
    tix = []
    for t, gid in enumerate(order):
        counts = gg.groups[gid].type_counts
        tix.append(np.asarray([lookup.get(name, unknown) for name in sorted(counts)
                               for _ in range(counts[name])], dtype=np.intp))
        sizes = sorted(gg.output_elem_counts(gid), reverse=True)[:shape_slots]
        shape[t, :len(sizes)] = np.log1p(sizes)
        for nb in list(gg.in_groups[gid]) + list(gg.out_groups[gid]):
            adj[t, nb % adj_slots] = 1.0
    return Features(order, tix, shape, adj)


def _sig(v):
    return 1.0 / (1.0 + np.exp(-v))


class Policy:
    """One parameter snapshot bound to one graph's features."""

    def __init__(self, flat, dims: Dims, feats: Features):
        self.dims, self.feats = dims, feats
        self.p = split_flat(flat, dims)

    # -- cell -------------------------------------------------------------------
    def _cell(self, w, b, x, h, c):
        H = self.dims.hidden
        xh = np.concatenate([x, h])
        pre = xh @ w + b
        gi, gf, go = _sig(pre[:H]), _sig(pre[H:2 * H]), _sig(pre[2 * H:3 * H])
        gg = np.tanh(pre[3 * H:])
        c2 = gf * c + gi * gg
        return o_tanh(go, c2), c2, (xh, gi, gf, go, gg, c, c2)

    @staticmethod
    def _cell_back(w, saved, dh, dc, n_x):
        xh, gi, gf, go, gg, c_in, c_out = saved
        th = np.tanh(c_out)
        d_o = dh * th
        dcell = dc + dh * go * (1.0 - th * th)
        d_pre = np.concatenate([(dcell * gg) * gi * (1.0 - gi), (dcell * c_in) * gf * (1.0 - gf),
                                d_o * go * (1.0 - go), (dcell * gi) * (1.0 - gg * gg)])
        d_xh = w @ d_pre
        return np.outer(xh, d_pre), d_pre, d_xh[:n_x], d_xh[n_x:], dcell * gf

    # -- forward ------------------------------------------------------------------
    def inputs(self):
        d, f, p = self.dims, self.feats, self.p
        rows = []
        for t in range(len(f.order)):
            rows.append(np.concatenate([p["type_table"][f.type_idx[t]].mean(axis=0), f.shape[t], f.adj[t]]))
        return np.array(rows).reshape(len(f.order), d.feat)

    def run(self, pick):
        """Encoder + attentional decoder; ``pick(t, probs)`` chooses each device."""
        d, p, order = self.dims, self.p, self.feats.order
        T, H, D = len(order), d.hidden, d.n_dev
        if T == 0:
            raise ValueError("cannot place an empty group sequence")
        x = self.inputs()
        h, c = np.zeros(H), np.zeros(H)
        enc_saved, enc = [], np.empty((T, H))
        for t in range(T):
            h, c, s = self._cell(p["w_enc"], p["b_enc"], x[t], h, c)
            enc_saved.append(s)
            enc[t] = h
        proj = enc @ p["w_att"].T
        steps, logp = [], 0.0
        placement = [0] * T
        row = D
        for t in range(T):
            h, c, s = self._cell(p["w_dec"], p["b_dec"], p["dev_table"][row], h, c)
            sc = proj @ h
            sc = sc - sc.max()
            att = np.exp(sc)
            att /= att.sum()
            hc = np.concatenate([h, att @ enc])
            u = hc @ p["w_out"]
            z = p["dev_table"][:D] @ u + p["b_out"]
            zs = z - z.max()
            lse = np.log(np.exp(zs).sum())
            probs = np.exp(zs - lse)
            k = int(pick(t, probs))
            logp += float(zs[k] - lse)
            steps.append((s, att, hc, u, probs, k, row))
            placement[order[t]] = k
            row = k
        return placement, logp, (x, enc_saved, enc, proj, steps)

    def sample(self, rng):
        D = self.dims.n_dev

        def pick(_t, probs):
            return min(int(np.searchsorted(np.cumsum(probs), rng.random(), side="right")), D - 1)

        return self.run(pick)

    def _forced(self, placement):
        if len(placement) != len(self.feats.order):
            raise ValueError(f"placement length {len(placement)} != sequence length {len(self.feats.order)}")
        for dv in placement:
            if not (0 <= dv < self.dims.n_dev):
                raise ValueError(f"device id {dv} out of range (D={self.dims.n_dev})")
        order = self.feats.order
        return self.run(lambda t, _p: placement[order[t]])

    def log_prob(self, placement) -> float:
        return self._forced(placement)[1]

    def step_probs(self, placement) -> np.ndarray:
        return np.stack([st[4] for st in self._forced(placement)[2][4]])

    # -- backward -----------------------------------------------------------------
    def grad(self, placement, tape=None) -> np.ndarray:
        if tape is None:
            tape = self._forced(placement)[2]
        d, p = self.dims, self.p
        H, D = d.hidden, d.n_dev
        x, enc_saved, enc, proj, steps = tape
        T = len(steps)
        g = {k: np.zeros(s) for k, s in d.shapes().items()}
        d_enc = np.zeros_like(enc)
        d_proj = np.zeros_like(proj)
        dh, dc = np.zeros(H), np.zeros(H)
        for t in reversed(range(T)):
            saved, att, hc, u, probs, k, row = steps[t]
            dz = -probs.copy()
            dz[k] += 1.0
            g["b_out"] += dz
            g["dev_table"][:D] += np.outer(dz, u)
            du = p["dev_table"][:D].T @ dz
            g["w_out"] += np.outer(hc, du)
            dhc = p["w_out"] @ du
            dh += dhc[:H]
            dctx = dhc[H:]
            datt = enc @ dctx
            d_enc += np.outer(att, dctx)
            dsc = att * (datt - att @ datt)
            d_proj += np.outer(dsc, hc[:H])
            dh += proj.T @ dsc
            dw, dpre, dx, dh, dc = self._cell_back(p["w_dec"], saved, dh, dc, d.dev_dim)
            g["w_dec"] += dw
            g["b_dec"] += dpre
            g["dev_table"][row] += dx
        g["w_att"] += d_proj.T @ enc
        d_enc += d_proj @ p["w_att"]
        dx_all = np.zeros_like(x)
        for t in reversed(range(T)):
            dh += d_enc[t]
            dw, dpre, dx, dh, dc = self._cell_back(p["w_enc"], enc_saved[t], dh, dc, d.feat)
            g["w_enc"] += dw
            g["b_enc"] += dpre
            dx_all[t] = dx
        for t in range(T):
            idx = self.feats.type_idx[t]
            np.add.at(g["type_table"], idx, dx_all[t, :d.type_dim] / len(idx))
        return join_flat(g)


def o_tanh(o, c):
    return o * np.tanh(c)
