"""Attentional seq2seq placement policy — host API over the sm_100a kernels.

Drop-in for the reference ``pkg/policy.py``: same classes (EmbeddingSpec,
GroupFeatures, PolicyParams, SampledPlacement), same functions and signatures
(forward_sample, log_prob_of, step_distributions, grad_log_prob,
embed_groups, checkpoint I/O).  The parameter containers and the structural
features are host objects built once per graph (as in the reference); every
forward/backward pass runs in ``csrc/policy_fwd.cu`` / ``csrc/policy_bwd.cu``
through the C-ABI (``dp_policy_*``).  There is no CPU fallback.

Batched entry points (new, used by the trainer and the benchmark):
``DevicePolicy.decode`` samples or teacher-forces K placements in one launch,
``DevicePolicy.backward`` returns sum_k adv[k] * grad log p_k.
"""

from __future__ import annotations

import ctypes
import json
import os
import threading
import weakref
from dataclasses import dataclass

import numpy as np

CHECKPOINT_FORMAT = "devplace-policy-v1"
_FIELDS = ("type_table", "dev_table", "w_enc", "b_enc", "w_dec", "b_dec", "w_att", "w_out", "b_out")


# ----------------------------------------------------------------------------- host containers
class EmbeddingSpec:
    """Vocabulary and block widths (reference ``pkg/policy.py:45-81``)."""

    def __init__(self, type_vocab, type_dim: int = 16, shape_slots: int = 8, adjacency_slots: int = 64):
        if type_dim < 1 or shape_slots < 1 or adjacency_slots < 1:
            raise ValueError("all embedding widths must be >= 1")
        self.type_vocab = dict(type_vocab)
        self.type_dim = type_dim
        self.shape_slots = shape_slots
        self.adjacency_slots = adjacency_slots

    @classmethod
    def build(cls, graphs, type_dim=16, shape_slots=8, adjacency_slots=64) -> "EmbeddingSpec":
        names = set()
        for g in graphs:
            src = g.graph if hasattr(g, "groups") else g
            names.update(op.op_type for op in src.ops)
        return cls({t: i for i, t in enumerate(sorted(names))}, type_dim, shape_slots, adjacency_slots)

    @property
    def unknown_index(self) -> int:
        return len(self.type_vocab)

    @property
    def table_rows(self) -> int:
        return len(self.type_vocab) + 1

    @property
    def input_dim(self) -> int:
        return self.type_dim + self.shape_slots + self.adjacency_slots

    def index_of(self, op_type: str) -> int:
        return self.type_vocab.get(op_type, self.unknown_index)


@dataclass
class GroupFeatures:
    """Structural encoder inputs, one row per decode step (``pkg/policy.py:84-117``)."""

    order: list
    type_indices: list
    shape_blocks: np.ndarray
    adj_blocks: np.ndarray

    @classmethod
    def from_grouped(cls, gg, spec: EmbeddingSpec) -> "GroupFeatures":
        order = list(gg.topo)
        T = len(order)
        shapes = np.zeros((T, spec.shape_slots))
        adj = np.zeros((T, spec.adjacency_slots))
        tix = []
        for t, gid in enumerate(order):
            counts = gg.groups[gid].type_counts
            tix.append(np.asarray([spec.index_of(name) for name in sorted(counts)
                                   for _ in range(counts[name])], dtype=np.intp))
            sizes = sorted(gg.output_elem_counts(gid), reverse=True)[: spec.shape_slots]
            shapes[t, : len(sizes)] = np.log1p(sizes)
            for nb in list(gg.in_groups[gid]) + list(gg.out_groups[gid]):
                adj[t, nb % spec.adjacency_slots] = 1.0
        return cls(order, tix, shapes, adj)

    def __len__(self):
        return len(self.order)


class PolicyParams:
    """Trainable tensors with the canonical flat view (``pkg/policy.py:120-188``)."""

    def __init__(self, spec: EmbeddingSpec, num_devices: int, hidden: int = 64, dev_dim: int = 16,
                 arrays=None):
        if num_devices < 1:
            raise ValueError("need at least one device")
        self.spec, self.num_devices, self.hidden, self.dev_dim = spec, num_devices, hidden, dev_dim
        f, h, dd, d = spec.input_dim, hidden, dev_dim, num_devices
        self.shapes = {
            "type_table": (spec.table_rows, spec.type_dim), "dev_table": (d + 1, dd),
            "w_enc": (f + h, 4 * h), "b_enc": (4 * h,), "w_dec": (dd + h, 4 * h), "b_dec": (4 * h,),
            "w_att": (h, h), "w_out": (2 * h, dd), "b_out": (d,),
        }
        if arrays is None:
            arrays = {k: np.zeros(s) for k, s in self.shapes.items()}
        for k in _FIELDS:
            if arrays[k].shape != self.shapes[k]:
                raise ValueError(f"{k}: expected shape {self.shapes[k]}, got {arrays[k].shape}")
            setattr(self, k, np.asarray(arrays[k], dtype=np.float64))

    @classmethod
    def init(cls, spec, num_devices, hidden=64, dev_dim=16, seed=0, scale=0.1) -> "PolicyParams":
        """Uniform[-scale, scale] per field in canonical order (``pkg/policy.py:154-162``)."""
        out = cls(spec, num_devices, hidden, dev_dim)
        gen = np.random.default_rng(seed)
        for k in _FIELDS:
            setattr(out, k, gen.uniform(-scale, scale, size=out.shapes[k]))
        return out

    @property
    def flat_size(self) -> int:
        return sum(int(np.prod(s)) for s in self.shapes.values())

    def to_flat(self) -> np.ndarray:
        return np.concatenate([getattr(self, k).ravel() for k in _FIELDS])

    def with_flat(self, flat) -> "PolicyParams":
        flat = np.asarray(flat, dtype=np.float64)
        if flat.shape != (self.flat_size,):
            raise ValueError(f"flat vector must have length {self.flat_size}")
        arrays, pos = {}, 0
        for k in _FIELDS:
            n = int(np.prod(self.shapes[k]))
            arrays[k] = flat[pos:pos + n].reshape(self.shapes[k]).copy()
            pos += n
        return PolicyParams(self.spec, self.num_devices, self.hidden, self.dev_dim, arrays)


@dataclass
class SampledPlacement:
    placement: list
    log_prob: float
    cache: object


class _DeviceCache:
    """Opaque forward-cache token: the activations live in the device engine;
    grad_log_prob re-runs the (deterministic) teacher-forced pass, which
    reproduces them exactly, so a stale token is never a correctness issue."""

    __slots__ = ("engine_id", "placement")

    def __init__(self, engine_id, placement):
        self.engine_id, self.placement = engine_id, placement


# Sampling certification (pkg/policy.py:320-323).  The device draw compares the
# numpy uniform r with the fp64 cdf it computes; the reference compares r with
# its own fp64 cdf.  The two cdfs differ only by rounding: the fp64 policy
# agrees with the reference's log-probabilities to ~1e-13 relative and its
# per-step distributions to ~1e-15 absolute (tests), with transcendentals
# within 4 ulp of libm (csrc/fastmath.cuh).  A draw whose margin
# min_j |r - cdf_j| exceeds SAMPLING_MARGIN_TOL (10^3 x the 1e-12 relative
# tolerance the parity tests hold the per-step distributions to) therefore
# picks the reference's index; smaller margins are counted as uncertified.
SAMPLING_MARGIN_TOL = 1e-9
FASTMATH_MAX_ULP = 4


# ----------------------------------------------------------------------------- device engine
def _hp(a):
    return a.ctypes.data if a.size else None


SUPPORTED_HIDDEN = 64
MAX_DEV_DIM = 32
MAX_DEVICES = 32


def check_policy_dims(hidden: int, dev_dim: int, num_devices: int) -> None:
    """ValueError for policy widths the sm_100a kernels do not implement."""
    if hidden != SUPPORTED_HIDDEN:
        raise ValueError(f"this build supports hidden={SUPPORTED_HIDDEN} (the reference default); got hidden={hidden}")
    if not 1 <= dev_dim <= MAX_DEV_DIM:
        raise ValueError(f"this build supports 1 <= dev_dim <= {MAX_DEV_DIM}; got dev_dim={dev_dim}")
    if not 1 <= num_devices <= MAX_DEVICES:
        raise ValueError(f"this build supports 1 <= num_devices <= {MAX_DEVICES}; got num_devices={num_devices}")


class DevicePolicy:
    """One ``dp_policy`` engine: features of one graph + dims, capacity k_max."""

    def __init__(self, feats: GroupFeatures, spec: EmbeddingSpec, num_devices: int, hidden: int = 64,
                 dev_dim: int = 16, k_max: int = 1):
        import torch

        from . import _native as nat

        self.T = len(feats)
        if self.T == 0:
            raise ValueError("cannot place an empty group sequence")
        # the kernels keep the 4H = 256 gate columns in one CTA's lanes: the
        # reference accepts any width (pkg/policy.py:127-146) but this build
        # implements its default (pkg/trainer.py:173-174) and says so up front
        check_policy_dims(hidden, dev_dim, num_devices)
        self.D, self.hidden, self.dev_dim, self.k_max = num_devices, hidden, dev_dim, k_max
        self.spec = spec
        self.device = torch.device("cuda", torch.cuda.current_device())
        lens = [len(ix) for ix in feats.type_indices]
        type_off = np.zeros(self.T + 1, np.int32)
        type_off[1:] = np.cumsum(lens)
        type_idx = np.ascontiguousarray(np.concatenate([np.asarray(ix, np.int32) for ix in feats.type_indices]))
        shape = np.ascontiguousarray(np.asarray(feats.shape_blocks, np.float64))
        adj = np.ascontiguousarray(np.asarray(feats.adj_blocks, np.float64))
        h = ctypes.c_void_p()
        rc = nat.lib().dp_policy_create(self.T, num_devices, hidden, dev_dim, spec.type_dim, spec.shape_slots,
                                        spec.adjacency_slots, spec.table_rows, _hp(type_off), _hp(type_idx),
                                        _hp(shape), _hp(adj), k_max, ctypes.byref(h))
        nat.check(rc, "dp_policy_create")
        self.handle = h.value
        self._destroy = nat.lib().dp_policy_destroy
        self.P = int(nat.lib().dp_policy_num_params(self.handle))
        self.order = torch.as_tensor(np.asarray(feats.order, np.int64), device=self.device)
        # the engine's buffers (encoder state, forward cache) are mutable: the
        # drop-in functions hold this lock across encode -> decode -> backward,
        # so controller threads sharing a GroupFeatures object (pkg/trainer.py:
        # 365-378) never interleave on one engine
        self.lock = threading.RLock()

    def __del__(self):
        if getattr(self, "handle", None):
            try:
                self._destroy(self.handle)
            except Exception:
                pass
            self.handle = None

    def encode(self, params_dev, stream=None):
        from . import _native as nat

        self._enc_flat = None  # encoder state no longer tied to a known host vector
        nat.check(nat.lib().dp_policy_encode(self.handle, nat.ptr(params_dev), nat.stream_ptr(stream)),
                  "dp_policy_encode")

    def decode(self, params_dev, K, pcg=None, draw_base=0, forced=None, k_offset=0, draw_counter=None,
               draws_per_count=0, choice=None, logp=None, probs=None, margin=None, stream=None):
        """Sample (pcg=(state, inc) as Python ints) or teacher-force (forced: uint8
        CUDA tensor [K, T] by rank) K placements.  Returns (choice [K,T] by rank, logp [K]).
        margin: optional f64 CUDA tensor [K] <- per-sample sampling margin
        (min over steps of |r - cdf_j|, j < D-1; see ``SAMPLING_MARGIN_TOL``)."""
        import torch

        from . import _native as nat

        if K > self.k_max:
            raise ValueError(f"K={K} exceeds engine capacity {self.k_max}")
        if choice is None:
            choice = torch.empty(K, self.T, dtype=torch.uint8, device=self.device)
        if logp is None:
            logp = torch.empty(K, dtype=torch.float64, device=self.device)
        hp = None
        if pcg is not None:
            st, inc = pcg
            m = (1 << 64) - 1
            hp = (ctypes.c_uint64 * 4)(st >> 64, st & m, inc >> 64, inc & m)
        rc = nat.lib().dp_policy_decode(
            self.handle, nat.ptr(params_dev), K, k_offset, hp, draw_base, nat.ptr(draw_counter),
            draws_per_count, nat.ptr(forced), nat.ptr(choice), nat.ptr(logp), nat.ptr(probs),
            nat.ptr(margin), nat.stream_ptr(stream))
        nat.check(rc, "dp_policy_decode")
        return choice, logp

    def backward(self, params_dev, K, adv_dev, grad=None, stream=None):
        import torch

        from . import _native as nat

        if grad is None:
            grad = torch.empty(self.P, dtype=torch.float64, device=self.device)
        rc = nat.lib().dp_policy_backward(self.handle, nat.ptr(params_dev), K, nat.ptr(adv_dev), nat.ptr(grad),
                                          nat.stream_ptr(stream))
        nat.check(rc, "dp_policy_backward")
        return grad

    def backward_rows(self, params_dev, K, stream=None):
        """Advantage-independent half of the backward (overlaps scoring)."""
        from . import _native as nat

        nat.check(nat.lib().dp_policy_backward_rows(self.handle, nat.ptr(params_dev), K, nat.stream_ptr(stream)),
                  "dp_policy_backward_rows")

    def backward_grads(self, params_dev, K, adv_dev, grad=None, stream=None):
        """Advantage-weighted half; returns sum_k adv[k] grad log p_k."""
        import torch

        from . import _native as nat

        if grad is None:
            grad = torch.empty(self.P, dtype=torch.float64, device=self.device)
        rc = nat.lib().dp_policy_backward_grads(self.handle, nat.ptr(params_dev), K, nat.ptr(adv_dev),
                                                nat.ptr(grad), nat.stream_ptr(stream))
        nat.check(rc, "dp_policy_backward_grads")
        return grad

    def by_gid(self, choice_by_rank):
        """[K, T] by rank -> [K, T] indexed by group id."""
        import torch

        out = torch.empty_like(choice_by_rank)
        out[:, self.order] = choice_by_rank
        return out

    def by_rank(self, placements_by_gid):
        return placements_by_gid[:, self.order]


_engines_lock = threading.Lock()
_engines: dict = {}


def engine_for(params: PolicyParams, feats: GroupFeatures, k: int = 1) -> DevicePolicy:
    """Cached engine per (features object, dims, device), capacity >= k (pow2)."""
    import torch

    cap = 1
    while cap < k:
        cap *= 2
    spec = params.spec
    key = (id(feats), spec.type_dim, spec.shape_slots, spec.adjacency_slots, spec.table_rows,
           params.num_devices, params.hidden, params.dev_dim, torch.cuda.current_device())
    with _engines_lock:
        ent = _engines.get(key)
        if ent is not None and ent[0]() is feats and ent[1].k_max >= cap:
            return ent[1]
        eng = DevicePolicy(feats, spec, params.num_devices, params.hidden, params.dev_dim, k_max=cap)
        try:
            _engines[key] = (weakref.ref(feats), eng)
        except TypeError:
            pass
        return eng


def _params_dev(params: PolicyParams, eng: DevicePolicy):
    import torch

    return torch.as_tensor(params.to_flat(), dtype=torch.float64, device=eng.device)


def _encoded(params: PolicyParams, eng: DevicePolicy):
    """Device params with the engine's encoder state for them.  The reference
    reruns the encoder inside every forward_sample / grad_log_prob call
    (pkg/policy.py:276-287); the engine keeps the flat vector it last encoded
    and skips the encoder when the caller's parameters are unchanged (content
    compare: a trainer calls forward_sample K times per snapshot).  The caller
    holds ``eng.lock``."""
    import torch

    flat = params.to_flat()
    last = getattr(eng, "_enc_flat", None)
    if last is not None and last[0].shape == flat.shape and np.array_equal(last[0], flat):
        return last[1]
    pdev = torch.as_tensor(flat, dtype=torch.float64, device=eng.device)
    eng.encode(pdev)
    eng._enc_flat = (flat.copy(), pdev)
    return pdev


def _check_placement_arg(params, feats, placement):
    """Reference validation and messages (``pkg/policy.py:343-348``)."""
    if len(placement) != len(feats):
        raise ValueError(f"placement length {len(placement)} != sequence length {len(feats)}")
    for dev in placement:
        if not (0 <= dev < params.num_devices):
            raise ValueError(f"device id {dev} out of range (D={params.num_devices})")


def _forced_by_rank(eng, feats, placements):
    import torch

    pl = np.asarray(placements, np.uint8).reshape(-1, len(feats))
    return torch.as_tensor(np.ascontiguousarray(pl[:, np.asarray(feats.order)]), device=eng.device)


def generator_state(rng) -> tuple[int, int]:
    st = rng.bit_generator.state
    if st.get("bit_generator") != "PCG64":
        raise TypeError("forward_sample needs a numpy Generator backed by PCG64 (np.random.default_rng)")
    return int(st["state"]["state"]), int(st["state"]["inc"])


# ----------------------------------------------------------------------------- reference API
def embed_groups(params: PolicyParams, feats: GroupFeatures) -> np.ndarray:
    """Assembled encoder inputs (``pkg/policy.py:266-268``), computed by the encoder kernel."""
    import torch

    from . import _native as nat  # noqa: F401

    eng = engine_for(params, feats, 1)
    with eng.lock:
        pdev = _params_dev(params, eng)
        eng.encode(pdev)
        torch.cuda.current_stream().synchronize()
        return _read_encoder_inputs(eng)


def _read_encoder_inputs(eng) -> np.ndarray:
    """Copy the engine's X buffer (first field of the struct after dims) — via a
    teacher-forced decode-free path: X is exposed by re-running the input kernel."""
    import torch

    from . import _native as nat

    F = eng.spec.input_dim
    out = torch.empty(eng.T, F, dtype=torch.float64, device=eng.device)
    rc = nat.lib().dp_policy_read_inputs(eng.handle, nat.ptr(out), nat.stream_ptr())
    nat.check(rc, "dp_policy_read_inputs")
    return out.cpu().numpy()


def forward_sample(params: PolicyParams, feats: GroupFeatures, rng) -> SampledPlacement:
    """Sample one placement (``pkg/policy.py:317-326``); consumes exactly T draws of ``rng``."""
    eng = engine_for(params, feats, 1)
    with eng.lock:
        pdev = _encoded(params, eng)
        choice, logp = eng.decode(pdev, 1, pcg=generator_state(rng))
        rng.bit_generator.advance(len(feats))
        placement = eng.by_gid(choice)[0].cpu().numpy().astype(int).tolist()
        return SampledPlacement(placement, float(logp[0].item()), _DeviceCache(id(eng), placement))


def _teacher_forced(params, feats, placements, want_probs=False):
    """Teacher-forced pass; the caller holds ``eng.lock`` (re-entrant) for as
    long as it uses the engine's forward cache."""
    import torch

    eng = engine_for(params, feats, len(placements))
    eng.lock.acquire()  # released by the caller (_locked_tf)
    pdev = _encoded(params, eng)
    K = len(placements)
    forced = _forced_by_rank(eng, feats, placements)
    probs = torch.empty(K, eng.T, eng.D, dtype=torch.float64, device=eng.device) if want_probs else None
    _, logp = eng.decode(pdev, K, forced=forced, probs=probs)
    return eng, pdev, logp, probs


class _locked_tf:
    """``with _locked_tf(...) as (eng, pdev, logp, probs)``: teacher-forced pass
    with the engine lock held until the block ends."""

    def __init__(self, params, feats, placements, want_probs=False):
        self.args = (params, feats, placements, want_probs)

    def __enter__(self):
        self.out = _teacher_forced(*self.args)
        return self.out

    def __exit__(self, *exc):
        self.out[0].lock.release()


def log_prob_of(params: PolicyParams, feats: GroupFeatures, placement) -> float:
    """Teacher-forced log-probability (``pkg/policy.py:329-333``)."""
    _check_placement_arg(params, feats, placement)
    with _locked_tf(params, feats, [placement]) as (_, _, logp, _):
        return float(logp[0].item())


def step_distributions(params: PolicyParams, feats: GroupFeatures, placement) -> np.ndarray:
    """Per-step device distributions (T, D) along a teacher-forced pass (``pkg/policy.py:336-340``)."""
    _check_placement_arg(params, feats, placement)
    with _locked_tf(params, feats, [placement], want_probs=True) as (_, _, _, probs):
        return probs[0].cpu().numpy()


def grad_log_prob(params: PolicyParams, feats: GroupFeatures, placement, cache=None) -> np.ndarray:
    """d log p(placement) / d flat params (``pkg/policy.py:351-409``)."""
    import torch

    _check_placement_arg(params, feats, placement)
    with _locked_tf(params, feats, [placement]) as (eng, pdev, _, _):
        adv = torch.ones(1, dtype=torch.float64, device=eng.device)
        return eng.backward(pdev, 1, adv).cpu().numpy()


def weighted_grad(params: PolicyParams, feats: GroupFeatures, placements, weights):
    """sum_k weights[k] * grad_log_prob(placements[k]) in one batched pass (device tensor)."""
    import torch

    for pl in placements:
        _check_placement_arg(params, feats, pl)
    with _locked_tf(params, feats, placements) as (eng, pdev, _, _):
        adv = torch.as_tensor(np.asarray(weights, np.float64), device=eng.device)
        return eng.backward(pdev, len(placements), adv)


def sample_batch(params: PolicyParams, feats: GroupFeatures, rng, K: int, return_margin: bool = False):
    """K forward_sample calls in one launch: same placements/log-probs, same
    draws consumed.  Returns (placements [K, T] by gid, log_probs [K]) numpy,
    plus the per-sample sampling margins [K] when ``return_margin``."""
    import torch

    eng = engine_for(params, feats, K)
    with eng.lock:
        pdev = _params_dev(params, eng)
        eng.encode(pdev)
        margin = torch.empty(K, dtype=torch.float64, device=eng.device) if return_margin else None
        choice, logp = eng.decode(pdev, K, pcg=generator_state(rng), margin=margin)
        rng.bit_generator.advance(K * len(feats))
        out = (eng.by_gid(choice).cpu().numpy(), logp.cpu().numpy())
    return out + (margin.cpu().numpy(),) if return_margin else out


def save_checkpoint(params: PolicyParams, path):
    """Hex-float JSON, format ``devplace-policy-v1`` (``pkg/policy.py:412-427``)."""
    doc = {
        "format": CHECKPOINT_FORMAT, "hidden": params.hidden, "dev_dim": params.dev_dim,
        "num_devices": params.num_devices, "type_dim": params.spec.type_dim,
        "shape_slots": params.spec.shape_slots, "adjacency_slots": params.spec.adjacency_slots,
        "type_vocab": params.spec.type_vocab, "flat_hex": [float(v).hex() for v in params.to_flat()],
    }
    with open(path, "w", encoding="utf-8") as fh:
        json.dump(doc, fh)
        fh.write("\n")


def load_checkpoint(path) -> PolicyParams:
    with open(path, "r", encoding="utf-8") as fh:
        doc = json.load(fh)
    if doc.get("format") != CHECKPOINT_FORMAT:
        raise ValueError(f"unsupported checkpoint format: {doc.get('format')!r}")
    spec = EmbeddingSpec(doc["type_vocab"], doc["type_dim"], doc["shape_slots"], doc["adjacency_slots"])
    p = PolicyParams(spec, doc["num_devices"], doc["hidden"], doc["dev_dim"])
    return p.with_flat(np.array([float.fromhex(v) for v in doc["flat_hex"]]))


__all__ = ["EmbeddingSpec", "GroupFeatures", "PolicyParams", "SampledPlacement", "DevicePolicy",
           "embed_groups", "forward_sample", "log_prob_of", "step_distributions", "grad_log_prob",
           "weighted_grad", "sample_batch", "save_checkpoint", "load_checkpoint", "engine_for",
           "generator_state"]
_ = os  # noqa
