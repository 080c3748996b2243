"""REINFORCE trainer — the batched hot path, device-resident.

Drop-in for the reference ``pkg/trainer.py`` (same names, signatures, log
format and determinism contract).  One update of one controller
(``run_controller`` body, pkg/trainer.py:271-308) is a fixed sequence of
sm_100a launches on one stream, with no host synchronisation:

  dp_policy_encode   encoder once per snapshot
  dp_policy_decode   K samples, PCG64 draws replayed from the controller stream
  dp_simulate_batch  K placements scored (event-exact simulator)
  dp_reinforce_epilogue  rewards, best, success-only, baseline, advantages
  dp_policy_backward sum_k adv_k * grad log p_k
  [NCCL all-reduce of the gradient when sharded over ranks]
  dp_adam_apply      finite check, Adam, version/update counters, log row

so the whole update can be captured once in a CUDA graph and replayed.
"""

from __future__ import annotations

import copy
import io
import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import policy as policy_mod
from .policy import EmbeddingSpec, GroupFeatures, PolicyParams
from .simulator import INFEASIBLE, SimReport, device_graph, simulate


def make_exchange(group):
    """The K-sharded exchange for a torch.distributed group: the library's own
    NCCL communicator when the group runs NCCL (one per process, captured in the
    update's CUDA graph), else torch.distributed host-staged (gloo)."""
    import os

    import torch.distributed as dist

    from .parallel import NcclExchange, TorchExchange

    if dist.get_backend(group) == "nccl" and os.environ.get("DP_EXCHANGE", "nccl") == "nccl":
        return NcclExchange.from_group(group)
    return TorchExchange(group)


# ----------------------------------------------------------------------------- reference types
@dataclass(frozen=True)
class RewardSpec:
    failing_signal: float

    def __post_init__(self):
        if not self.failing_signal > 0:
            raise ValueError("failing_signal must be > 0")


def suggest_failing_signal(gg, topo) -> float:
    """2 x sqrt(total cost / slowest rate) (``pkg/trainer.py:46-53``)."""
    slowest = min(d.compute_rate for d in topo.devices)
    return 2.0 * math.sqrt(gg.total_compute_cost() / slowest)


def validate_failing_signal(spec: RewardSpec, gg, topo):
    slowest = min(d.compute_rate for d in topo.devices)
    bound = math.sqrt(gg.total_compute_cost() / slowest)
    if spec.failing_signal <= bound:
        raise ValueError(
            f"failing_signal {spec.failing_signal} does not exceed the "
            f"slowest-single-device bound sqrt({gg.total_compute_cost()}/{slowest}) = {bound}")


def reward_of(measurement: float, spec: RewardSpec) -> float:
    """``pkg/trainer.py:66-72`` (scalar; the batched form runs in dp_reinforce_epilogue)."""
    if measurement == INFEASIBLE:
        return spec.failing_signal
    if not math.isfinite(measurement) or measurement <= 0:
        raise ValueError(f"measurement must be positive and finite, got {measurement}")
    return math.sqrt(measurement)


@dataclass
class BaselineState:
    value: float
    decay: float = 0.9
    initialized_from_failing_signal: bool = False

    def update(self, mean_reward: float):
        self.value = self.decay * self.value + (1.0 - self.decay) * mean_reward


def _state_tensor(device, baseline=0.0):
    import torch

    from . import _native as nat

    st = torch.zeros(nat.TRAIN_STATE_WORDS, dtype=torch.float64, device=device)
    st[0] = baseline
    st[2] = math.inf
    return st


def _state_read(st) -> dict:
    from . import _native as nat

    raw = st.cpu()
    f = raw.numpy()
    i = raw.view(dtype=__import__("torch").int64).numpy()
    out = {}
    for k, name in enumerate(nat.TRAIN_STATE_FIELDS):
        out[name] = float(f[k]) if k < 3 else int(i[k])
    return out


class ParameterStore:
    """Authoritative flat parameters + Adam moments on the GPU (``pkg/trainer.py:87-131``).

    ``snapshot()`` returns a host copy; ``apply(g)`` runs the device Adam
    kernel.  The controller loop uses the device tensors directly."""

    def __init__(self, flat, learning_rate=1e-3, beta1=0.9, beta2=0.999, epsilon=1e-8, device=None,
                 max_steps: int = 1 << 16):
        import threading

        import torch

        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.params = torch.as_tensor(np.array(flat, dtype=np.float64), device=self.device).clone()
        self.m = torch.zeros_like(self.params)
        self.v = torch.zeros_like(self.params)
        self.learning_rate, self.beta1, self.beta2, self.epsilon = learning_rate, beta1, beta2, epsilon
        self.state = _state_tensor(self.device)
        self.flag = torch.zeros(1, dtype=torch.int32, device=self.device)
        self._bias_cap = 0
        self.bias = None
        self._old_bias = []
        self._ensure_bias(max_steps)
        self._lock = threading.Lock()
        self._scratch_log = torch.zeros(8, dtype=torch.float64, device=self.device)

    def _ensure_bias(self, steps):
        import torch

        if steps <= self._bias_cap:
            return
        tab = np.empty(2 * steps)
        for t in range(1, steps + 1):  # Python float pow, as ParameterStore.apply computes it
            tab[2 * (t - 1)] = 1.0 - self.beta1 ** t
            tab[2 * (t - 1) + 1] = 1.0 - self.beta2 ** t
        if self.bias is not None:
            # a captured CUDA graph may still hold the old table's address (its
            # launches carry their own t_cap and flag error 3 beyond it): keep it alive
            self._old_bias.append(self.bias)
        self.bias = torch.as_tensor(tab, device=self.device)
        self._bias_cap = steps

    @property
    def version(self) -> int:
        return _state_read(self.state)["version"]

    @property
    def rejected(self) -> int:
        return _state_read(self.state)["rejected"]

    def snapshot(self):
        with self._lock:
            return self.params.cpu().numpy().copy(), self.version

    def adam(self, grad, log=None, log_cap=0, stream=None, state=None):
        """Enqueue dp_adam_apply (grad = advantage-weighted sum; /n_used inside).
        ``state``: the applying controller's state (n_used, update, log row);
        the store's own counters (adam_t, version, rejected) live in ``self.state``."""
        from . import _native as nat

        rc = nat.lib().dp_adam_apply(
            self.params.numel(), nat.ptr(self.params), nat.ptr(self.m), nat.ptr(self.v), nat.ptr(grad),
            nat.ptr(self.bias), self._bias_cap, self.learning_rate, self.beta1, self.beta2, self.epsilon,
            nat.ptr(state if state is not None else self.state), nat.ptr(self.state), nat.ptr(self.flag),
            nat.ptr(log if log is not None else self._scratch_log), log_cap, nat.stream_ptr(stream))
        nat.check(rc, "dp_adam_apply")

    def apply(self, gradient) -> int:
        """Adam step in the descent direction; returns the store version."""
        import torch

        g = np.asarray(gradient, dtype=np.float64)
        with self._lock:
            if g.shape != tuple(self.params.shape):
                raise ValueError(f"gradient length {g.shape} != parameter length {tuple(self.params.shape)}")
            st = _state_read(self.state)
            self._ensure_bias(st["adam_t"] + 1)
            self.state.view(torch.int64)[7] = 1  # n_used = 1: apply() receives the final gradient
            self.adam(torch.as_tensor(g, device=self.device))
            return _state_read(self.state)["version"]


def apply_adam(store: ParameterStore, gradient) -> int:
    return store.apply(gradient)


def reinforce_update(params: PolicyParams, feats: GroupFeatures, samples, rewards, baseline: BaselineState):
    """Advantage-weighted mean of log-prob gradients (``pkg/trainer.py:138-154``),
    one batched teacher-forced pass + one backward on the GPU."""
    if not samples:
        return None
    b = baseline.value
    w = [r - b for r in rewards]
    g = policy_mod.weighted_grad(params, feats, [s.placement for s in samples], w)
    g = (g / len(samples)).cpu().numpy()
    baseline.update(float(np.mean(rewards)))
    return g


@dataclass
class TrainerConfig:
    k: int = 4
    total_updates: int = 200
    success_only_after: int = 5000
    learning_rate: float = 1e-3
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_epsilon: float = 1e-8
    seed: int = 0
    controllers: int = 1
    workers_per_controller: int | None = None
    baseline_decay: float = 0.9
    failing_signal: float | None = None
    noise_sigma: float = 0.0
    measure_steps: int = 10
    hidden: int = 64
    dev_dim: int = 16
    type_dim: int = 16
    shape_slots: int = 8
    adjacency_slots: int = 64
    init_scale: float = 0.1
    # new (not in the reference): GPUs the K samples are sharded over in this
    # one process.  None = every visible GPU (the largest count dividing k);
    # a tuple of CUDA device indices = exactly those (repeats share a GPU).
    devices: tuple | None = None

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if self.success_only_after < 0:
            raise ValueError("success_only_after must be >= 0")


@dataclass
class LogRow:
    update_index: int
    controller_id: int
    store_version: int
    mean_r: float
    baseline: float
    best_r: float
    n_feasible: int
    n_used: int
    wall_ms: float

    CSV_HEADER = "update_index,controller_id,store_version,mean_R,baseline,best_R,n_feasible_of_K,wall_ms"

    def csv_line(self, include_wall: bool = True) -> str:
        cells = [str(self.update_index), str(self.controller_id), str(self.store_version),
                 repr(self.mean_r), repr(self.baseline), repr(self.best_r), str(self.n_feasible)]
        if include_wall:
            cells.append(f"{self.wall_ms:.3f}")
        return ",".join(cells)


def log_to_csv(rows, include_wall: bool = True) -> str:
    header = LogRow.CSV_HEADER if include_wall else LogRow.CSV_HEADER.rsplit(",", 1)[0]
    buf = io.StringIO()
    buf.write(header + "\n")
    for row in rows:
        buf.write(row.csv_line(include_wall) + "\n")
    return buf.getvalue()


@dataclass
class TrainResult:
    best_placement: list | None
    best_report: SimReport | None
    log: list
    final_params: np.ndarray
    store_versions: int
    rejected_updates: int
    # sampling certificate (DeviceController.sampling_certificate; new field)
    sampling: dict | None = None

    @property
    def found_feasible(self) -> bool:
        return self.best_placement is not None

    @property
    def best_makespan(self):
        return self.best_report.makespan_seconds if self.best_report else None


@dataclass
class _TrainTask:
    gg: object
    topo: object
    feats: GroupFeatures
    template: PolicyParams
    reward_spec: RewardSpec
    config: TrainerConfig


@dataclass
class _ControllerResult:
    rows: list = field(default_factory=list)
    best_r: float = math.inf
    best_placement: list | None = None
    sampling: dict | None = None


def policy_template(gg, topo, config: TrainerConfig) -> PolicyParams:
    spec = EmbeddingSpec.build([gg], type_dim=config.type_dim, shape_slots=config.shape_slots,
                               adjacency_slots=config.adjacency_slots)
    return PolicyParams.init(spec, topo.num_devices, hidden=config.hidden, dev_dim=config.dev_dim,
                             seed=config.seed, scale=config.init_scale)


# ----------------------------------------------------------------------------- device controller
class DeviceController:
    """One controller's REINFORCE loop on one GPU (or one rank's shard of K).

    ``world=(rank, size, comm)`` shards the K samples (rank r owns samples
    [r*K/size, (r+1)*K/size)); per update the ranks all-gather one small
    record each (scores + the shard's best candidate row, parallel.py) so every
    rank replays the reference's sequential best / baseline logic
    bit-identically, and all-reduce the gradient.  ``comm``: a
    torch.distributed group (NCCL -> the library's own NCCL communicator,
    captured in the update's CUDA graph; gloo -> host-staged), an exchange
    object (parallel.NcclExchange / TorchExchange), or ``"external"`` (a
    multi-device runner issues the collectives between the step's phases)."""

    def __init__(self, task: _TrainTask, store: ParameterStore, seed_seq, controller_id: int = 0,
                 world=None, log_cap: int | None = None, shared: bool = False):
        """``shared``: several controllers share ``store`` (f1): this controller
        keeps its own state (baseline, best, update counter, log) and samples
        from a private parameter snapshot taken by the runner; the store's
        counters (adam_t, version, rejected) stay in ``store.state``."""
        import torch

        cfg = task.config
        self.task, self.store, self.cid = task, store, controller_id
        self.device = store.device
        from .parallel import shard

        self.rank, self.size, comm = world if world is not None else (0, 1, None)
        K = cfg.k
        self.K = K
        self.k_offset, self.K_local = shard(K, self.rank, self.size)
        self.xchg = None
        if comm == "external":
            self.exchanged = True
        else:
            if hasattr(comm, "all_gather"):
                self.xchg = comm
            elif comm is not None and self.size > 1:
                self.xchg = make_exchange(comm)
            self.exchanged = self.xchg is not None
        tmpl = task.template
        self.eng = policy_mod.DevicePolicy(task.feats, tmpl.spec, tmpl.num_devices, tmpl.hidden, tmpl.dev_dim,
                                           k_max=self.K_local)
        self.dg = device_graph(task.gg, task.topo)
        self.T = len(task.feats)
        sample_seq, noise_seq = seed_seq.spawn(2)
        self.rng = np.random.default_rng(sample_seq)
        self.pcg = policy_mod.generator_state(self.rng)
        self.log_cap = log_cap if log_cap is not None else cfg.total_updates
        store._ensure_bias(cfg.total_updates * max(1, cfg.controllers) + 1)
        self.shared = shared
        # every controller keeps its own state (baseline, best, update counter,
        # n_used, error); the store's counters (adam_t, version, rejected) stay in
        # store.state, so a store that already applied updates continues its
        # version numbering and Adam step as the reference's does
        self.state = _state_tensor(store.device)
        self.params_src = torch.empty_like(store.params) if shared else store.params
        st = self.state
        st[0] = task.reward_spec.failing_signal
        st[2] = math.inf
        dev = self.device
        T = self.T
        self.choice = torch.zeros(self.K_local, T, dtype=torch.uint8, device=dev)
        self.logp = torch.zeros(self.K_local, dtype=torch.float64, device=dev)
        # sampling certification: per-sample margin of the last update and the
        # running minimum / count of samples below policy.SAMPLING_MARGIN_TOL
        self.margin = torch.full((self.K_local,), math.inf, dtype=torch.float64, device=dev)
        self.margin_min = torch.full((1,), math.inf, dtype=torch.float64, device=dev)
        self.n_uncertified = torch.zeros(1, dtype=torch.int64, device=dev)
        self.sim_local = None
        self.adv = torch.zeros(self.K_local, dtype=torch.float64, device=dev)
        self.grad = torch.zeros(store.params.numel(), dtype=torch.float64, device=dev)
        self.best_choice = torch.zeros(T, dtype=torch.uint8, device=dev)
        self.log = torch.full((max(1, self.log_cap) * 8,), math.nan, dtype=torch.float64, device=dev)
        if self.exchanged:
            from . import _native as nat

            rb = int(nat.lib().dp_exchange_record_bytes(self.K_local, T))
            self.rec = torch.zeros(rb, dtype=torch.uint8, device=dev)
            self.recs = torch.zeros(self.size * rb, dtype=torch.uint8, device=dev)
            self.mk_all = torch.zeros(K, dtype=torch.float64, device=dev)
            self.fe_all = torch.zeros(K, dtype=torch.uint8, device=dev)
            self.rows_all = torch.zeros(self.size, T, dtype=torch.uint8, device=dev)
        self.measure_ok = cfg.measure_steps >= 2
        # measurement noise (f2): the factor rows of every update, drawn up front
        # from the controller's noise stream exactly as the reference does
        self.noise = None
        if cfg.noise_sigma > 0.0 and self.measure_ok and cfg.total_updates > 0:
            tab = noise_factor_table(noise_seq, K, cfg.total_updates, cfg.noise_sigma, cfg.measure_steps)
            self.noise = torch.as_tensor(tab, device=dev).contiguous()
        self.updates_done = 0
        self._graph = None
        self.side = torch.cuda.Stream(device=dev)

    # one update, enqueue-only (capturable)
    def step(self, stream=None, marks=None, apply: bool = True):
        """Enqueue one update.  ``marks``: optional callable(name) recording a
        CUDA event at each phase boundary (bench.py phase timing).
        ``apply=False`` stops before the Adam step (the shared-store runner
        orders the controllers' applies itself)."""
        self.phase_sample(stream, marks)
        if self.xchg is not None:
            (marks or (lambda _n: None))("exchange")
            self.xchg.all_gather(self.recs, self.rec, stream=stream)
        self.phase_score(stream, marks)
        if self.xchg is not None:
            (marks or (lambda _n: None))("allreduce")
            self.xchg.all_reduce_sum(self.grad, stream=stream)
        if apply:
            (marks or (lambda _n: None))("adam")
            self.apply(stream)
        (marks or (lambda _n: None))("end")

    def phase_sample(self, stream=None, marks=None):
        """Encode, sample this shard, score it (the advantage-independent half of
        the backward overlaps on a side stream); sharded: pack the exchange record."""
        import torch

        from . import _native as nat

        mark = marks or (lambda _name: None)
        cfg = self.task.config
        p = self.params_src
        state = self.state
        main = stream if stream is not None else torch.cuda.current_stream()
        mark("encode")
        self.eng.encode(p, stream)
        mark("decode")
        self.eng.decode(p, self.K_local, pcg=self.pcg, draw_base=0, k_offset=self.k_offset,
                        draw_counter=state.view(torch.int64)[3:4], draws_per_count=self.K * self.T,
                        choice=self.choice, logp=self.logp, margin=self.margin, stream=stream)
        mark("simulate")
        # the advantage-independent half of the backward runs on a side stream
        # while the placements are scored
        self.side.wait_stream(main)
        self.eng.backward_rows(p, self.K_local, stream=self.side)
        # sampling certificate, off the rows pass's path
        nat.check(nat.lib().dp_margin_accumulate(self.K_local, nat.ptr(self.margin), policy_mod.SAMPLING_MARGIN_TOL,
                                                 nat.ptr(self.margin_min), nat.ptr(self.n_uncertified),
                                                 nat.stream_ptr(stream)), "dp_margin_accumulate")
        self.sim_local = self.dg.simulate(self.choice, by_rank=True, stream=stream, out=self.sim_local)
        mk, fe = self.sim_local["makespan"], self.sim_local["feasible"]
        if not self.measure_ok:
            fe.zero_()  # measure() raises for steps < 2 -> every worker reports INFEASIBLE
        if self.noise is not None:
            nat.check(nat.lib().dp_apply_measurement_noise(
                self.K_local, self.k_offset, self.K, nat.ptr(mk), nat.ptr(fe), nat.ptr(self.noise),
                self.noise.shape[0], self.noise.shape[2], nat.ptr(state), nat.stream_ptr(stream)),
                "dp_apply_measurement_noise")
        if self.exchanged:
            nat.check(nat.lib().dp_exchange_pack(self.K_local, self.T, nat.ptr(mk), nat.ptr(fe),
                                                 nat.ptr(self.choice), nat.ptr(self.rec), nat.stream_ptr(stream)),
                      "dp_exchange_pack")

    def phase_score(self, stream=None, marks=None):
        """Rewards / best / baseline / advantages over all K (after the exchange),
        then the advantage-weighted backward."""
        import torch

        from . import _native as nat

        mark = marks or (lambda _name: None)
        cfg = self.task.config
        main = stream if stream is not None else torch.cuda.current_stream()
        if self.exchanged:
            nat.check(nat.lib().dp_exchange_unpack(self.size, self.K_local, self.T, nat.ptr(self.recs),
                                                   nat.ptr(self.mk_all), nat.ptr(self.fe_all),
                                                   nat.ptr(self.rows_all), nat.stream_ptr(stream)),
                      "dp_exchange_unpack")
            mk, fe, ch, div = self.mk_all, self.fe_all, self.rows_all, self.K_local
        else:
            mk, fe, ch, div = self.sim_local["makespan"], self.sim_local["feasible"], self.choice, 1
        mark("epilogue")
        rc = nat.lib().dp_reinforce_epilogue(
            self.K, self.T, nat.ptr(mk), nat.ptr(fe), nat.ptr(ch), div, self.task.reward_spec.failing_signal,
            cfg.baseline_decay, cfg.success_only_after, self.k_offset, self.K_local, nat.ptr(self.state),
            nat.ptr(self.adv), nat.ptr(self.best_choice), nat.ptr(self.log), self.log_cap, self.cid,
            nat.stream_ptr(stream))
        nat.check(rc, "dp_reinforce_epilogue")
        mark("backward")
        # backward_grads waits on the rows pass itself (its attention sums start
        # as soon as the attention backward is done, beside the LSTM backward)
        self.eng.backward_grads(self.params_src, self.K_local, self.adv, grad=self.grad, stream=stream)
        main.wait_stream(self.side)

    def apply(self, stream=None):
        """This controller's Adam step on the (possibly shared) store."""
        self.store.adam(self.grad, log=self.log, log_cap=self.log_cap, stream=stream, state=self.state)

    def capture(self):
        """Capture one update in a CUDA graph (after one eager warm-up update)."""
        import gc

        import torch

        # no destructor (cudaFree) may run while the stream is capturing
        gc.collect()
        gc.disable()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.step()
        finally:
            gc.enable()
        self._graph = g
        return g

    def run(self, updates: int, use_graph: bool = True, wall=None):
        """Run ``updates`` updates; returns per-update wall ms (device-synchronised)."""
        import torch

        walls = []
        for _ in range(updates):
            t0 = time.perf_counter()
            if use_graph and self._graph is not None:
                self._graph.replay()
            else:
                self.step()
            if wall is not None:
                torch.cuda.current_stream().synchronize()
                walls.append((time.perf_counter() - t0) * 1e3)
            self.updates_done += 1
        return walls

    def check_errors(self):
        st = _state_read(self.state)
        if st["error"] == 2:
            raise RuntimeError("measurement-noise table exhausted (more updates than total_updates)")
        if st["error"] == 3:
            raise RuntimeError("Adam bias-correction table exhausted (more updates than the store's max_steps)")
        if st["error"]:
            raise ValueError("measurement must be positive and finite (a feasible placement has makespan <= 0)")
        return st

    def rows(self, walls=None) -> list:
        arr = self.log.cpu().numpy().reshape(-1, 8)
        out = []
        for u in range(min(self.updates_done, self.log_cap)):
            r = arr[u]
            out.append(LogRow(int(r[0]), int(r[1]), int(r[2]), float(r[3]), float(r[4]), float(r[5]),
                              int(r[6]), int(r[7]), float(walls[u]) if walls else 0.0))
        return out

    def sampling_certificate(self) -> dict:
        """Minimum sampling margin over every sample drawn so far and the number
        of samples with a draw closer than policy.SAMPLING_MARGIN_TOL to a cdf
        boundary (those indices are not certified equal to the reference's);
        over all ranks when sharded."""
        mm = self.margin_min.clone()
        nu = self.n_uncertified.to(dtype=mm.dtype)
        if self.xchg is not None:
            self.xchg.all_reduce_min(mm)
            self.xchg.all_reduce_sum(nu)
            import torch

            torch.cuda.current_stream().synchronize()
        return {"min_margin": float(mm.item()), "tol": policy_mod.SAMPLING_MARGIN_TOL,
                "uncertified_samples": int(nu.item()), "fastmath_max_ulp": policy_mod.FASTMATH_MAX_ULP}

    def best(self):
        st = _state_read(self.state)
        if not math.isfinite(st["best_r"]):
            return math.inf, None
        pl = self.eng.by_gid(self.best_choice.view(1, -1))[0].cpu().numpy().astype(int).tolist()
        return st["best_r"], pl


def _noise_rows(args):
    seeds, sigma, steps = args
    out = np.empty((len(seeds), steps - 1))
    for i, sd in enumerate(seeds):
        out[i] = np.exp(sigma * np.random.default_rng(sd).standard_normal(steps))[1:]
    return out


def noise_factor_table(noise_seq, K: int, updates: int, sigma: float, steps: int) -> np.ndarray:
    """[updates, K, steps-1] lognormal factors of the reference's noisy measure()
    (``pkg/trainer.py:262, 277`` seeds; ``pkg/simulator.py:221-223`` factors):
    seeds come sequentially from the controller's noise stream, each
    measurement's factors from ``default_rng(seed).standard_normal(steps)``.
    Large tables fan the per-seed generators out over host processes."""
    rng = np.random.default_rng(noise_seq)
    seeds = [int(rng.integers(1 << 62)) for _ in range(updates * K)]
    n = len(seeds)
    if n > 20000:
        import concurrent.futures as cf
        import os

        w = max(1, min(32, len(os.sched_getaffinity(0))))
        chunk = (n + w - 1) // w
        with cf.ProcessPoolExecutor(w) as ex:
            parts = list(ex.map(_noise_rows, [(seeds[i:i + chunk], sigma, steps) for i in range(0, n, chunk)]))
        flat = np.concatenate(parts)
    else:
        flat = _noise_rows((seeds, sigma, steps))
    return flat.reshape(updates, K, steps - 1)


class ConcurrentRunner:
    """Several DeviceControllers advancing together, one CUDA stream each, all
    captured into one CUDA graph per round.

    * shared store (f1, ``TrainerConfig.controllers > 1``, pkg/trainer.py:
      365-378): every round all controllers snapshot the same store version
      (device copies on the launching stream), sample / score / differentiate
      concurrently on their own streams, then apply in controller order — a
      deterministic member of the reference's asynchronous interleavings
      (oracle.trainer.run_multi restates it);
    * independent stores (C4 mixed batch, ``train_many``): each controller's
      whole update, Adam included, runs on its own stream."""

    def __init__(self, ctls, shared_store: ParameterStore | None = None, concurrent: bool = True):
        """``concurrent=False`` enqueues the controllers one after another on
        the launching stream (required when their steps issue collectives on
        one communicator: every rank must see the same collective order)."""
        import torch

        self.ctls, self.store = list(ctls), shared_store
        self.concurrent = concurrent
        self.streams = [torch.cuda.Stream(device=c.device) for c in self.ctls] if concurrent else None
        self._graph = None

    def step(self):
        import torch

        main = torch.cuda.current_stream()
        if self.store is not None:
            for c in self.ctls:
                c.params_src.copy_(self.store.params)
        if not self.concurrent:
            for c in self.ctls:
                c.step(stream=main, apply=self.store is None)
            if self.store is not None:
                for c in self.ctls:
                    c.apply(main)
            return
        for c, s in zip(self.ctls, self.streams):
            s.wait_stream(main)
            with torch.cuda.stream(s):
                c.step(stream=s, apply=self.store is None)
        for s in self.streams:
            main.wait_stream(s)
        if self.store is not None:
            for c in self.ctls:
                c.apply(main)

    def capture(self):
        import gc

        import torch

        gc.collect()
        gc.disable()
        try:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self.step()
        finally:
            gc.enable()
        self._graph = g
        return g

    def run(self, updates: int, use_graph: bool = True, wall: bool = False):
        import torch

        walls = []
        for _ in range(updates):
            t0 = time.perf_counter()
            if use_graph and self._graph is not None:
                self._graph.replay()
            else:
                self.step()
            if wall:
                torch.cuda.current_stream().synchronize()
                walls.append((time.perf_counter() - t0) * 1e3)
            for c in self.ctls:
                c.updates_done += 1
        return walls

    def train(self, updates: int):
        """First round eager, then one captured graph replayed."""
        import torch

        walls = []
        if updates > 0:
            walls += self.run(1, use_graph=False, wall=True)
        if updates > 1:
            self.capture()
            walls += self.run(updates - 1, use_graph=True, wall=True)
        torch.cuda.current_stream().synchronize()
        for c in self.ctls:
            c.check_errors()
        return walls


def _result_of(task, store, ctls, walls) -> "TrainResult":
    res = []
    for c in ctls:
        r = _ControllerResult(rows=c.rows(walls), sampling=c.sampling_certificate())
        r.best_r, r.best_placement = c.best()
        res.append(r)
    rows = sorted([row for r in res for row in r.rows], key=lambda r: (r.controller_id, r.update_index))
    best = min(res, key=lambda r: r.best_r)
    best_pl = list(best.best_placement) if best.best_placement is not None else None
    best_report = simulate(task.gg, task.topo, best_pl) if best_pl is not None else None
    final, _ = store.snapshot()
    return TrainResult(best_placement=best_pl, best_report=best_report, log=rows, final_params=final,
                       store_versions=store.version, rejected_updates=store.rejected,
                       sampling=_merge_certs([r.sampling for r in res]))


def _merge_certs(certs):
    certs = [c for c in certs if c]
    if not certs:
        return None
    out = dict(certs[0])
    out["min_margin"] = min(c["min_margin"] for c in certs)
    out["uncertified_samples"] = sum(c["uncertified_samples"] for c in certs)
    return out


def train_many(jobs) -> list:
    """Train several independent tasks at once (config C4, the mixed batch):
    ``jobs`` = [(graph, topo, TrainerConfig), ...], each with its own
    parameters, store, baseline and RNG streams, advanced together on their own
    CUDA streams (one graph replay per round).  Each result equals
    ``train(graph, topo, config)`` run alone."""
    from .graph import coalesce_sole_consumers

    prepared = []
    for graph, topo, config in jobs:
        config = config or TrainerConfig()
        if config.controllers != 1:
            raise ValueError("train_many: each job runs one controller")
        gg = graph if hasattr(graph, "groups") else coalesce_sole_consumers(graph)
        task = _make_task(gg, topo, config)
        store = ParameterStore(task.template.to_flat(), learning_rate=config.learning_rate,
                               beta1=config.adam_beta1, beta2=config.adam_beta2, epsilon=config.adam_epsilon,
                               max_steps=config.total_updates + 1)
        seq = np.random.SeedSequence(config.seed).spawn(1)[0]
        prepared.append((task, store, DeviceController(task, store, seq, 0)))
    ups = {t.config.total_updates for t, _, _ in prepared}
    if len(ups) == 1:
        runner = ConcurrentRunner([c for _, _, c in prepared])
        walls = runner.train(ups.pop())
        return [_result_of(t, s, [c], walls) for t, s, c in prepared]
    # different lengths: each job on its own (still device-resident and graph-replayed)
    out = []
    for t, s, c in prepared:
        r = run_controller(0, s, t, None, ctl=c)
        out.append(_result_of(t, s, [c], [row.wall_ms for row in r.rows]))
    return out


def _make_task(gg, topo, config: TrainerConfig) -> _TrainTask:
    template = policy_template(gg, topo, config)
    feats = GroupFeatures.from_grouped(gg, template.spec)
    failing = config.failing_signal
    if failing is None:
        failing = suggest_failing_signal(gg, topo)
    reward_spec = RewardSpec(failing)
    validate_failing_signal(reward_spec, gg, topo)
    return _TrainTask(gg, topo, feats, template, reward_spec, config)


def run_controller(controller_id: int, store: ParameterStore, task: _TrainTask, seed_seq,
                   world=None, ctl=None) -> _ControllerResult:
    """``pkg/trainer.py:256-309`` on the device (CUDA-graph replay after update 0).

    ``world=(rank, size, group)`` runs this rank's K-shard (parallel.py); with
    NCCL the collectives are captured in the update's graph, with a
    host-staged (gloo) exchange the step runs eagerly."""
    import torch

    cfg = task.config
    if ctl is None:
        ctl = DeviceController(task, store, seed_seq, controller_id, world=world)
    use_graph = ctl.xchg is None or ctl.xchg.capturable
    walls = []
    if cfg.total_updates > 0:
        walls += ctl.run(1, use_graph=False, wall=True)
    if cfg.total_updates > 1:
        if use_graph:
            ctl.capture()
        walls += ctl.run(cfg.total_updates - 1, use_graph=use_graph, wall=True)
    torch.cuda.current_stream().synchronize()
    ctl.check_errors()
    res = _ControllerResult(rows=ctl.rows(walls), sampling=ctl.sampling_certificate())
    res.best_r, res.best_placement = ctl.best()
    return res


class MultiDeviceRunner:
    """One process drives G GPUs (a plain ``train()`` call
    uses every visible device).  Rank r (device ``devices[r]``) owns samples
    [r*K/G, (r+1)*K/G) with its own replicated parameter store; one update is
    the controllers' phases interleaved across devices with the two
    collectives in between (NCCL, one communicator per device from
    ``ncclCommInitAll``, each call group-wrapped; or device copies when every
    rank shares one GPU — parallel.LocalGroup).  The whole round — every
    device's kernels and both collectives — is captured once (one CUDA graph
    per device) and replayed."""

    def __init__(self, task: _TrainTask, config: TrainerConfig, devices, seed_seq):
        import torch

        from .parallel import LocalGroup, NcclExchange, NcclGroup

        self.devices = [int(d) for d in devices]
        G = len(self.devices)
        distinct = sorted(set(self.devices))
        if len(distinct) not in (1, G):
            raise ValueError(f"devices {self.devices}: either all distinct or all the same GPU")
        self.shared_gpu = len(distinct) == 1 and G > 1
        self.task, self.config = task, config
        self.streams, self.stores, self.ctls = [], [], []
        seed0 = copy.deepcopy(seed_seq)
        for r, d in enumerate(self.devices):
            with torch.cuda.device(d):
                s = torch.cuda.Stream(device=d) if (r == 0 or not self.shared_gpu) else self.streams[0]
                self.streams.append(s)
                st = ParameterStore(task.template.to_flat(), learning_rate=config.learning_rate,
                                    beta1=config.adam_beta1, beta2=config.adam_beta2, epsilon=config.adam_epsilon,
                                    device=torch.device("cuda", d), max_steps=config.total_updates + 1)
                self.stores.append(st)
                # every rank replays the same controller streams: spawn from a copy
                # (SeedSequence.spawn advances its child counter)
                self.ctls.append(DeviceController(task, st, copy.deepcopy(seed0), 0, world=(r, G, "external")))
        if self.shared_gpu:
            self.comm = LocalGroup(G)
        else:
            self.comm = NcclGroup(NcclExchange.init_all(self.devices), self.streams)
        self._graphs = None
        torch.cuda.synchronize(self.devices[0])

    def _each(self, fn):
        import torch

        for c, d, s in zip(self.ctls, self.devices, self.streams):
            with torch.cuda.device(d), torch.cuda.stream(s):
                fn(c, s)

    def step(self):
        import torch

        for d, s in zip(self.devices, self.streams):  # order after prior default-stream work
            with torch.cuda.device(d):
                s.wait_stream(torch.cuda.current_stream(d))
        self._each(lambda c, s: c.phase_sample(s))
        with torch.cuda.device(self.devices[0]), torch.cuda.stream(self.streams[0]):
            self.comm.all_gather([(c.recs, c.rec) for c in self.ctls])
        self._each(lambda c, s: c.phase_score(s))
        with torch.cuda.device(self.devices[0]), torch.cuda.stream(self.streams[0]):
            self.comm.all_reduce_sum([c.grad for c in self.ctls])
        self._each(lambda c, s: c.apply(s))
        for d, s in zip(self.devices, self.streams):
            with torch.cuda.device(d):
                torch.cuda.current_stream(d).wait_stream(s)

    def capture(self):
        import gc

        import torch

        gc.collect()
        gc.disable()
        devs = self.devices[:1] if self.shared_gpu else self.devices
        graphs = [torch.cuda.CUDAGraph() for _ in devs]
        try:
            for g, d, s in zip(graphs, devs, self.streams):
                with torch.cuda.device(d), torch.cuda.stream(s):
                    g.capture_begin(capture_error_mode="relaxed")
            self._each(lambda c, s: c.phase_sample(s))
            with torch.cuda.device(self.devices[0]), torch.cuda.stream(self.streams[0]):
                self.comm.all_gather([(c.recs, c.rec) for c in self.ctls])
            self._each(lambda c, s: c.phase_score(s))
            with torch.cuda.device(self.devices[0]), torch.cuda.stream(self.streams[0]):
                self.comm.all_reduce_sum([c.grad for c in self.ctls])
            self._each(lambda c, s: c.apply(s))
            for g, d, s in zip(graphs, devs, self.streams):
                with torch.cuda.device(d), torch.cuda.stream(s):
                    g.capture_end()
        finally:
            gc.enable()
        self._graphs = list(zip(graphs, devs, self.streams))

    def replay(self):
        import torch

        for g, d, s in self._graphs:
            with torch.cuda.device(d):
                s.wait_stream(torch.cuda.current_stream(d))
                with torch.cuda.stream(s):
                    g.replay()
                torch.cuda.current_stream(d).wait_stream(s)

    def run(self, updates, use_graph=True):
        import torch

        walls = []
        for _ in range(updates):
            t0 = time.perf_counter()
            if use_graph and self._graphs is not None:
                self.replay()
            else:
                self.step()
            for d in sorted(set(self.devices)):
                torch.cuda.synchronize(d)
            walls.append((time.perf_counter() - t0) * 1e3)
            for c in self.ctls:
                c.updates_done += 1
        return walls

    def train(self, updates):
        walls = []
        if updates > 0:
            walls += self.run(1, use_graph=False)
        if updates > 1:
            self.capture()
            walls += self.run(updates - 1, use_graph=True)
        for c in self.ctls:
            c.check_errors()
        return walls

    def result(self, walls) -> "TrainResult":
        import torch

        c0 = self.ctls[0]
        with torch.cuda.device(self.devices[0]):
            rows = sorted(c0.rows(walls), key=lambda r: (r.controller_id, r.update_index))
            best_r, best_pl = c0.best()
            final, _ = self.stores[0].snapshot()
            certs = []
            for c, d in zip(self.ctls, self.devices):
                with torch.cuda.device(d):
                    certs.append(c.sampling_certificate())
            best_report = simulate(self.task.gg, self.task.topo, best_pl) if best_pl is not None else None
        return TrainResult(best_placement=best_pl, best_report=best_report, log=rows, final_params=final,
                           store_versions=self.stores[0].version, rejected_updates=self.stores[0].rejected,
                           sampling=_merge_certs(certs))


def _auto_devices(config: TrainerConfig):
    """Devices a plain train() shards over: the configured tuple, or every
    visible GPU (the largest count that divides k)."""
    import torch

    if config.devices is not None:
        return tuple(int(d) for d in config.devices)
    n = torch.cuda.device_count()
    G = max(g for g in range(1, max(1, n) + 1) if config.k % g == 0)
    return tuple(range(G)) if G > 1 else (torch.cuda.current_device(),)


def train(graph, topo, config: TrainerConfig | None = None, *, group=None) -> TrainResult:
    """Train the policy; return the best feasible placement ever measured
    (``pkg/trainer.py:341-393``).

    Without ``group`` the K samples are sharded over ``config.devices`` (by
    default every visible GPU, the largest count dividing k) inside this one
    process (MultiDeviceRunner; NCCL).  ``group``: optional torch.distributed
    process group; every rank calls train() with the same arguments and owns
    K/size of the samples (one GPU per rank).  Every rank
    returns the same result.  ``controllers > 1`` (f1) runs on one GPU."""
    from .graph import coalesce_sole_consumers

    config = config or TrainerConfig()
    gg = graph if hasattr(graph, "groups") else coalesce_sole_consumers(graph)
    task = _make_task(gg, topo, config)
    C = config.controllers
    root = np.random.SeedSequence(config.seed)
    seqs = root.spawn(C)
    devices = _auto_devices(config) if group is None and C == 1 else None
    if devices is not None and len(devices) > 1:
        # one process, every GPU: K sharded over the devices (MultiDeviceRunner)
        runner = MultiDeviceRunner(task, config, devices, seqs[0])
        return runner.result(runner.train(config.total_updates))
    if devices is not None:
        import torch

        torch.cuda.set_device(devices[0])
    store = ParameterStore(task.template.to_flat(), learning_rate=config.learning_rate, beta1=config.adam_beta1,
                           beta2=config.adam_beta2, epsilon=config.adam_epsilon,
                           max_steps=config.total_updates * C + 1)
    if C > 1:
        # f1: C controllers over one device-resident store (ConcurrentRunner)
        if group is not None:
            raise NotImplementedError("multi-controller training with K sharded over ranks")
        ctls = [DeviceController(task, store, seqs[c], c, shared=True) for c in range(C)]
        walls = ConcurrentRunner(ctls, store).train(config.total_updates)
        return _result_of(task, store, ctls, walls)
    world = None
    if group is not None:
        import torch.distributed as dist

        world = (dist.get_rank(group), dist.get_world_size(group), group)
    res = run_controller(0, store, task, seqs[0], world=world)
    rows = sorted(res.rows, key=lambda r: (r.controller_id, r.update_index))
    best_pl = list(res.best_placement) if res.best_placement is not None else None
    best_report = simulate(gg, topo, best_pl) if best_pl is not None else None
    final, _ = store.snapshot()
    return TrainResult(best_placement=best_pl, best_report=best_report, log=rows, final_params=final,
                       store_versions=store.version, rejected_updates=store.rejected, sampling=res.sampling)
