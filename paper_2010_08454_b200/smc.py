"""Host orchestration of the SMC bootstrap particle filter (K4 init, K5 scan, K6 resample).

The engine has no reference counterpart (SPEC.md:455 lists SMC/particle methods as a
non-goal); its semantics are SURVEY.md §8(a) a17 / Appendix A D6 and are restated bit for bit
by oracle/cuppl_oracle.c (or_smc_*).

Per time step t, on every rank r (one process per GPU):
  1. all-reduce MAX of the max log-weight key  (NCCL; skipped for one rank)
  2. K5 scan: quantised weights, rank-local segment offsets, rank record {T_r, s1_r, s2_r}
  3. all-gather of the 32-byte rank records    (NCCL; skipped for one rank)
  4. K6 resample(t) -> population t+1: the outputs whose ancestors live on rank r are produced
     by rank r and stored straight into their owner's buffers (peer pointers).
With several processes the x / lw buffers live in cudaMalloc'd arenas whose CUDA-IPC handles are
all-gathered once, so every rank holds a table of the peers' buffers (NVLink peer stores).
`local_world=R` runs R virtual ranks in one process on one GPU (same kernels, collectives done
with tensor ops) — it exercises the multi-rank arithmetic without a second GPU.
"""

from __future__ import annotations

import ctypes as C
import math
from dataclasses import dataclass, field

import numpy as np

from . import _native as N
from . import _nvtx
from .dists import alias_table
from .errors import AllZeroWeightError, InferRuntimeError
from .models import HiddenMarkovModel
from .rng import key_of, seed_of

INT32_MIN = -(2**31)


def key_to_float(k: int) -> float:
    """Inverse of the kernels' monotone float->int key (f2key)."""
    k = int(k) & 0xFFFFFFFF
    if k & 0x80000000:
        k ^= 0x7FFFFFFF
    return float(np.array([k], dtype=np.uint32).view(np.float32)[0])


@dataclass
class SmcResult:
    """Outcome of run_smc. Arrays are indexed by time step t = 0..T-1."""

    n_particles: int
    log_z: float
    log_z_steps: np.ndarray
    ess: np.ndarray
    max_log_weight: np.ndarray
    total_weight: np.ndarray          # integer weight totals T_t (exact)
    filtering: dict = field(default_factory=dict)   # t -> normalised state histogram
    filtering_int: dict = field(default_factory=dict)  # t -> integer weights per state
    states: object = None             # final population (tensor per rank) and log-weights
    log_weights: object = None
    ancestors: list = field(default_factory=list)   # per step (when recorded)


def rank_boundaries(n: int, world: int) -> list[int]:
    """Global index of each rank's first particle; multiples of 16 (16-byte state stores,
    Philox blocks of 4 outputs)."""
    if n < 16 * world:
        raise ValueError("n_particles must be >= 16 * world_size")
    n16 = n // 16
    return [16 * (n16 * q // world) for q in range(world)] + [n]


class _DevArray:
    """Zero-copy torch view of library-allocated device memory (__cuda_array_interface__)."""

    def __init__(self, ptr: int, n: int, typestr: str):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None}


def _align(v: int) -> int:
    return (v + 255) & ~255


class _Arena:
    """x[2] (and anc[2]) of one rank in one cudaMalloc'd arena shareable by CUDA IPC."""

    def __init__(self, n: int, with_anc: bool, device):
        import torch

        self.n = n
        self.off = {}
        o = 0
        # xch: the peer-exchange mailboxes and flags of both phases (cuppl_peer_exchange):
        # [mbox A: 32 x 64 B][flags A: 32 x u64][mbox B][flags B]
        for name, size in ((("x0", n), ("x1", n)) + ((("anc0", 8 * n), ("anc1", 8 * n)) if with_anc else ())
                           + (("xch", 2 * (32 * 64 + 32 * 8)),)):
            self.off[name] = o
            o += _align(size)
        self.bytes = o
        p = C.c_void_p()
        N.check(N.lib().cuppl_arena_alloc(o, C.byref(p)), "arena_alloc")
        self.base = p.value
        with torch.cuda.device(device):
            self.x = [torch.as_tensor(_DevArray(self.base + self.off[f"x{i}"], n, "|u1"), device=device)
                      for i in range(2)]
            xb = 2 * (32 * 64 + 32 * 8)
            torch.as_tensor(_DevArray(self.base + self.off["xch"], xb, "|u1"), device=device).zero_()
            self.anc = ([torch.as_tensor(_DevArray(self.base + self.off[f"anc{i}"], n, "<i8"), device=device)
                         for i in range(2)] if with_anc else None)

    def handle(self) -> bytes:
        h = (C.c_char * 64)()
        N.check(N.lib().cuppl_ipc_handle(C.c_void_p(self.base), h), "ipc_handle")
        return bytes(h)

    def __del__(self):  # pragma: no cover - interpreter teardown order
        try:
            N.lib().cuppl_arena_free(C.c_void_p(self.base))
        except Exception:
            pass


class _Rank:
    """Device state of one rank."""

    def __init__(self, runner, r: int):
        import torch

        self.r = r
        dev = runner.device
        lo, hi = runner.bounds[r], runner.bounds[r + 1]
        self.lo, self.n = lo, hi - lo
        if runner.multiprocess:
            self.arena = _Arena(self.n, runner.record_ancestors, dev)
            self.x, self.anc = self.arena.x, self.arena.anc
        else:
            self.arena = None
            self.x = [torch.empty(self.n, dtype=torch.uint8, device=dev) for _ in range(2)]
            self.anc = ([torch.empty(self.n, dtype=torch.int64, device=dev) for _ in range(2)]
                        if runner.record_ancestors else None)
        ws = N.lib().cuppl_smc_workspace_bytes(self.n)
        self.ws = torch.empty(int(ws), dtype=torch.uint8, device=dev)
        self.m_key = torch.full((runner.T,), INT32_MIN, dtype=torch.int32, device=dev)
        self.rec = torch.zeros((runner.T, 4), dtype=torch.int64, device=dev)
        self.stats = torch.zeros((runner.T, 2), dtype=torch.float64, device=dev)


class SmcRunner:
    def __init__(self, model: HiddenMarkovModel, n_particles: int, rng, *, group=None, device=None,
                 record_ancestors: bool = False, hist_steps=None, local_world: int | None = None,
                 steps: int | None = None, graph: bool = False, exchange: str = "auto"):
        import torch

        if not isinstance(model, HiddenMarkovModel):
            raise InferRuntimeError(f"no SMC kernel for {type(model).__name__}")
        if model.n_states > 256:
            raise InferRuntimeError("SMC kernels store the state in one byte: n_states <= 256")
        self.model = model
        self.N = int(n_particles)
        if self.N >= 2**31:
            raise InferRuntimeError("n_particles must be < 2^31 (u64 weight totals, u32 comb)")
        self.key = key_of(rng)
        self.seed = seed_of(rng)
        self.T = int(steps or model.T)
        if self.T > model.T:
            raise ValueError("steps exceeds the number of observations")
        self.record_ancestors = record_ancestors
        self.device = device or torch.device("cuda", torch.cuda.current_device())
        self.group = group
        self.local = local_world is not None
        if self.local:
            self.world, self.rank = int(local_world), 0
            self.ranks_here = list(range(self.world))
        else:
            from .infer import _world

            self.rank, self.world = _world(group)
            self.ranks_here = [self.rank]
        self.multiprocess = self.world > 1 and not self.local
        # multi-process exchanges: "peer" = cuppl_peer_exchange over the IPC-mapped arenas (device
        # only, graph-capturable), "collective" = torch.distributed (NCCL / gloo)
        if exchange not in ("auto", "peer", "collective"):
            raise ValueError("exchange must be 'auto', 'peer' or 'collective'")
        self.peer = self.multiprocess and (exchange == "peer" or (exchange == "auto" and self.world <= 32))
        if self.peer and self.world > 32:
            raise InferRuntimeError("peer exchange supports up to 32 ranks")
        self.bounds = rank_boundaries(self.N, self.world)
        S = model.n_states
        aliasA = np.array([alias_table(list(model.A[s])) for s in range(S)], dtype=np.uint64)
        alias0 = np.array(alias_table(list(model.pi0)), dtype=np.uint64)
        dev = self.device
        self.aliasA = torch.tensor(aliasA.reshape(-1).view(np.int64), device=dev)
        self.alias0 = torch.tensor(alias0.view(np.int64), device=dev)
        self.mu = np.ascontiguousarray(model.mu, dtype=np.float32)
        sd = float(model.sd)
        self.cm = N.SmcModel()
        self.cm.n_states = S
        self.cm.inv_sd = float(np.float32(1.0 / sd))
        self.cm.c = float(np.float32(-math.log(sd) - 0.5 * math.log(2 * math.pi)))
        self.cm.alias_trans = self.aliasA.data_ptr()
        self.cm.alias_init = self.alias0.data_ptr()
        self.cm.mu = self.mu.ctypes.data
        self.ys = np.ascontiguousarray(model.ys, dtype=np.float32)
        self.hist_steps = sorted(set(hist_steps if hist_steps is not None else [self.T - 1]))
        self.ranks = [_Rank(self, r) for r in self.ranks_here]
        self.hist = {t: torch.zeros((len(self.ranks), S), dtype=torch.int64, device=dev)
                     for t in self.hist_steps}
        self.rank_begin = torch.tensor(self.bounds, dtype=torch.int64, device=dev)
        self.gathered = torch.zeros((self.T, self.world, 4), dtype=torch.int64, device=dev)
        # destination pointer tables per ping-pong parity: x_out / lw_out / anc_out [world]
        self._peers = []
        if self.multiprocess:
            xps, aps = self._exchange_arenas()
            if self.peer:
                self.epoch = torch.zeros(2, dtype=torch.int64, device=dev)
                self.xstatus = torch.zeros(1, dtype=torch.int32, device=dev)
        self._tables = {}
        for par in (0, 1):
            if self.multiprocess:
                xp = xps[par]
                ap = aps[par] if record_ancestors else None
            else:
                xp = [rk.x[par].data_ptr() for rk in self.ranks]
                ap = [rk.anc[par].data_ptr() for rk in self.ranks] if record_ancestors else None
            self._tables[par] = (torch.tensor(xp, dtype=torch.int64, device=dev),
                                 torch.tensor(ap, dtype=torch.int64, device=dev) if ap else None)
        self.ancestors = []
        self._pending_anc = None
        self.cur = 0
        self.k6_events = None  # list of (start, end) CUDA events per K6 launch when profiling
        self.k6_every = 1      # time every k-th K6 launch only (fewer event nodes in a graph)
        # CUDA graph of the whole run (init + T steps): one process, no ancestor snapshots (their
        # host-side list cannot be replayed). The Philox key then lives in device memory
        # (cuppl_smc_model.key_dev), so one capture serves every reseed.
        self.use_graph = bool(graph) and (not self.multiprocess or self.peer) and not record_ancestors
        self.key_dev = None
        if self.use_graph:
            import torch

            self.key_dev = torch.zeros(1, dtype=torch.int64, device=dev)
            self.cm.key_dev = self.key_dev.data_ptr()
        self._graph = None
        self._graph_cur = 0
        self._capturing = False
        self.t_next = 0  # next population to scan (eager runs; see advance / snapshot)

    # ------------------------------------------------------------------ collectives -------
    def _exchange_arenas(self):
        """All-gather (IPC handle, offsets) of every rank's arena and map the peers'."""
        import torch.distributed as dist

        me = self.ranks[0].arena
        info = (me.handle(), me.off)
        allinfo = [None] * self.world
        dist.all_gather_object(allinfo, info, group=self.group)
        bases = []
        for q, (h, off) in enumerate(allinfo):
            if q == self.rank:
                bases.append((me.base, off))
                continue
            p = C.c_void_p()
            hb = (C.c_char * 64).from_buffer_copy(h)
            N.check(N.lib().cuppl_ipc_open(hb, C.byref(p)), "ipc_open")
            self._peers.append(p.value)
            bases.append((p.value, off))
        import torch

        self.peer_bases = torch.tensor([b for b, _ in bases], dtype=torch.int64, device=self.device)
        self.xch_off = me.off["xch"]
        xs = [[b + o[f"x{par}"] for b, o in bases] for par in (0, 1)]
        an = ([[b + o[f"anc{par}"] for b, o in bases] for par in (0, 1)] if self.record_ancestors else None)
        return xs, an

    def close(self):
        """Unmap peer arenas (the local arena is freed with the runner)."""
        for p in self._peers:
            N.lib().cuppl_ipc_close(C.c_void_p(p))
        self._peers = []

    def _backend(self) -> str:
        import torch.distributed as dist

        return dist.get_backend(self.group)

    def _allreduce_max(self, t: int):
        if self.world == 1:
            return
        import torch

        if self.local:
            m = torch.stack([rk.m_key[t] for rk in self.ranks]).max()
            for rk in self.ranks:
                rk.m_key[t].copy_(m)
        elif self.peer:
            v = self.ranks[0].m_key[t:t + 1]
            self._peer_exchange(v, 4, 0, max_out=v)
        else:
            import torch.distributed as dist

            v = self.ranks[0].m_key[t:t + 1]
            if self._backend() == "nccl":
                dist.all_reduce(v, op=dist.ReduceOp.MAX, group=self.group)
            else:  # gloo (tests): host round trip, also a barrier after this rank's K6
                h = v.cpu()
                dist.all_reduce(h, op=dist.ReduceOp.MAX, group=self.group)
                v.copy_(h)

    def _allgather(self, t: int):
        import torch

        if self.local or self.world == 1:
            for i, rk in enumerate(self.ranks):
                self.gathered[t, rk.r].copy_(rk.rec[t])
        elif self.peer:
            self._peer_exchange(self.ranks[0].rec[t], 32, 1, gather_out=self.gathered[t])
        else:
            import torch.distributed as dist

            if self._backend() == "nccl":
                dist.all_gather_into_tensor(self.gathered[t].view(-1), self.ranks[0].rec[t], group=self.group)
            else:
                h = torch.empty(self.world * 4, dtype=torch.int64)
                dist.all_gather_into_tensor(h, self.ranks[0].rec[t].cpu(), group=self.group)
                self.gathered[t].view(-1).copy_(h)

    PEER_TIMEOUT_NS = 60_000_000_000

    def _peer_exchange(self, src, nbytes: int, phase: int, max_out=None, gather_out=None):
        """cuppl_peer_exchange: phase 0 = MAX of the stabiliser keys, phase 1 = the rank records."""
        mbox = self.xch_off + phase * (32 * 64 + 32 * 8)
        N.check(N.lib().cuppl_peer_exchange(N.ptr(src), nbytes, N.ptr(self.peer_bases), mbox, mbox + 32 * 64,
                                            self.rank, self.world, N.ptr(self.epoch[phase:phase + 1]),
                                            N.ptr(max_out), N.ptr(gather_out), N.ptr(self.xstatus),
                                            self.PEER_TIMEOUT_NS, N.stream_ptr(self.device)), "peer_exchange")

    def _gather_stats(self) -> np.ndarray:
        import torch

        if self.local or self.world == 1:
            return torch.stack([rk.stats for rk in self.ranks]).cpu().numpy()
        import torch.distributed as dist

        if self._backend() == "nccl":
            out = torch.empty((self.world, self.T, 2), dtype=torch.float64, device=self.device)
            dist.all_gather_into_tensor(out.view(-1), self.ranks[0].stats.view(-1), group=self.group)
        else:
            out = torch.empty((self.world, self.T, 2), dtype=torch.float64)
            dist.all_gather_into_tensor(out.view(-1), self.ranks[0].stats.view(-1).cpu(), group=self.group)
        return out.cpu().numpy()

    # ------------------------------------------------------------------ steps -------------
    def reseed(self, rng):
        """Reuse the runner's buffers for a new run with another generator."""
        self.key = key_of(rng)
        self.seed = seed_of(rng)
        self.ancestors = []
        self._pending_anc = None

    def init(self):
        self.t_next = 0
        L = N.lib()
        st = N.stream_ptr(self.device)
        for h in self.hist.values():
            h.zero_()
        for rk in self.ranks:  # per-step maxima are atomicMax targets: a rerun starts from scratch
            rk.m_key.fill_(INT32_MIN)
        for rk in self.ranks:
            N.check(L.cuppl_smc_init(C.byref(self.cm), rk.n, rk.lo, self.key, float(self.ys[0]),
                                     N.ptr(rk.x[0]), N.ptr(rk.m_key[0:1]), N.ptr(rk.ws), rk.ws.numel(), st),
                    "smc_init", seed=self.seed)
        self.cur = 0

    def step(self, t: int):
        """Scan population t and (t < T-1) resample/propagate it to t+1."""
        L = N.lib()
        st = N.stream_ptr(self.device)
        self._allreduce_max(t)  # also the barrier after every rank's K6(t - 1) peer stores
        self._snapshot_ancestors()
        h = self.hist.get(t)
        with _nvtx.phase("smc.scan"):
            self._scan(t, h, L, st)
        with _nvtx.phase("smc.allgather"):
            self._allgather(t)
        if t + 1 >= self.T:
            with _nvtx.phase("smc.fold"):
                for rk in self.ranks:
                    N.check(L.cuppl_smc_fold(rk.n, N.ptr(rk.stats[t]), N.ptr(rk.ws), rk.ws.numel(), st),
                            "smc_fold", seed=self.seed, step=t)
            return
        with _nvtx.phase("smc.resample"):
            self._resample(t, L, st)

    def _scan(self, t, h, L, st):
        for i, rk in enumerate(self.ranks):
            N.check(L.cuppl_smc_scan(C.byref(self.cm), rk.n, float(self.ys[t]), N.ptr(rk.x[self.cur]),
                                     N.ptr(rk.m_key[t:t + 1]), None if h is None else N.ptr(h[i]),
                                     N.ptr(rk.rec[t]), N.ptr(rk.ws), rk.ws.numel(), st),
                    "smc_scan", seed=self.seed, step=t)

    def _resample(self, t, L, st):
        nxt = 1 - self.cur
        xt, at = self._tables[nxt]
        ev = None
        if self.k6_events is not None and t % self.k6_every == 0:
            import torch

            ext = self._capturing  # inside a graph: event-record nodes that time every replay
            ev = (torch.cuda.Event(enable_timing=True, external=ext),
                  torch.cuda.Event(enable_timing=True, external=ext))
            ev[0].record()
        for rk in self.ranks:
            N.check(L.cuppl_smc_resample(
                C.byref(self.cm), rk.n, self.N, self.key, t, rk.r, self.world, float(self.ys[t]),
                float(self.ys[t + 1]), N.ptr(rk.x[self.cur]), N.ptr(rk.m_key[t:t + 1]),
                N.ptr(self.gathered[t]), N.ptr(self.rank_begin), N.ptr(xt),
                None if at is None else N.ptr(at), N.ptr(rk.m_key[t + 1:t + 2]), N.ptr(rk.stats[t]),
                N.ptr(rk.ws), rk.ws.numel(), st), "smc_resample", seed=self.seed, step=t)
        if ev is not None:
            ev[1].record()
            self.k6_events.append(ev)
        if self.record_ancestors:
            self._pending_anc = nxt  # complete only after the next collective (peer stores)
        self.cur = nxt
        self.t_next = t + 1

    def log_weights(self, rk):
        """Per-particle log-weights of the current population (tabulated per state)."""
        import torch

        lw = torch.empty(rk.n, dtype=torch.float32, device=self.device)
        N.check(N.lib().cuppl_smc_log_weights(C.byref(self.cm), float(self.ys[self.T - 1]),
                                              N.ptr(rk.x[self.cur]), rk.n, N.ptr(lw),
                                              N.stream_ptr(self.device)), "smc_log_weights")
        return lw

    def _snapshot_ancestors(self):
        if self._pending_anc is not None:
            self.ancestors.append([rk.anc[self._pending_anc].clone() for rk in self.ranks])
            self._pending_anc = None

    def run(self) -> SmcResult:
        self.launch()
        return self.result()

    def launch(self):
        """Enqueue a whole run (init + T steps) on the current stream: replay of the captured
        graph in graph mode, else step by step."""
        if not self.use_graph:
            self.init()
            for t in range(self.T):
                self.step(t)
            self._snapshot_ancestors()
            return
        import torch

        self.key_dev.fill_(int(np.uint64(self.key).view(np.int64)))
        if self._graph is None:
            self._capture()
        with _nvtx.phase("smc.graph_replay"):
            self._graph.replay()
        self.cur = self._graph_cur

    def _capture(self):
        import torch

        torch.cuda.synchronize(self.device)
        g = torch.cuda.CUDAGraph()
        self._capturing = True
        try:
            with torch.cuda.graph(g, capture_error_mode="relaxed"):
                self.init()
                for t in range(self.T):
                    self.step(t)
        finally:
            self._capturing = False
        self._graph = g
        self._graph_cur = self.cur

    # ------------------------------------------------------------------ checkpoint -------
    def advance(self, until: int):
        """Eager run of populations [t_next, until) (init first when nothing ran yet)."""
        if self.use_graph:
            raise InferRuntimeError("advance/snapshot need an eager runner (graph=False)")
        if self.t_next == 0:
            self.init()
        for t in range(self.t_next, min(until, self.T)):
            self.step(t)
        if until >= self.T:
            self.t_next = self.T
            self._snapshot_ancestors()

    def snapshot(self) -> dict:
        """Host copy of the run state between steps: the current population, the per-step
        records / maxima / statistics / histograms so far and the scan workspace. Philox is
        counter-based, so (key, t_next) is the whole generator state."""
        import torch

        if self.use_graph or self.multiprocess:
            raise InferRuntimeError("snapshots are taken from eager single-process runners")
        torch.cuda.synchronize(self.device)
        self._snapshot_ancestors()
        return {"n": self.N, "T": self.T, "world": self.world, "key": self.key, "seed": self.seed,
                "t_next": self.t_next, "x": [rk.x[self.cur].cpu() for rk in self.ranks],
                "m_key": [rk.m_key.cpu() for rk in self.ranks], "rec": [rk.rec.cpu() for rk in self.ranks],
                "stats": [rk.stats.cpu() for rk in self.ranks], "ws": [rk.ws.cpu() for rk in self.ranks],
                "gathered": self.gathered.cpu(), "hist": {t: h.cpu() for t, h in self.hist.items()},
                "ancestors": [[a.cpu() for a in step] for step in self.ancestors]}

    def restore(self, snap: dict):
        """Load a snapshot into this runner (same model, population size, steps and ranks);
        resume() then continues exactly where the snapshot was taken."""
        if (snap["n"], snap["T"], snap["world"]) != (self.N, self.T, self.world) or self.use_graph:
            raise InferRuntimeError("snapshot does not match this runner (n, steps, ranks, eager)")
        if set(snap["hist"]) != set(self.hist):
            raise InferRuntimeError("snapshot histogram steps differ from this runner's")
        self.key, self.seed, self.t_next = snap["key"], snap["seed"], snap["t_next"]
        self.cur = 0
        self._pending_anc = None
        for i, rk in enumerate(self.ranks):
            rk.x[0].copy_(snap["x"][i])
            rk.m_key.copy_(snap["m_key"][i])
            rk.rec.copy_(snap["rec"][i])
            rk.stats.copy_(snap["stats"][i])
            rk.ws.copy_(snap["ws"][i])
        self.gathered.copy_(snap["gathered"])
        for t, h in snap["hist"].items():
            self.hist[t].copy_(h)
        self.ancestors = [[a.to(self.device) for a in step] for step in snap["ancestors"]]

    def resume(self) -> SmcResult:
        """Run the remaining steps and return the result of the whole run."""
        self.advance(self.T)
        return self.result()

    def k6_ms(self) -> float:
        """Sum of the recorded K6 launch durations (after a synchronize)."""
        return sum(a.elapsed_time(b) for a, b in self.k6_events or [])

    def result(self) -> SmcResult:
        if self.peer and int(self.xstatus.item()):
            raise InferRuntimeError("peer exchange timed out (a rank did not reach the step)", seed=self.seed)
        g = self.gathered.cpu().numpy().view(np.uint64)
        mk = self.ranks[0].m_key.cpu().numpy()
        Tt = g[:, :, 0].sum(axis=1)
        stats = self._gather_stats()  # [world, T, 2]
        s1 = np.zeros(self.T)
        s2 = np.zeros(self.T)
        for q in range(self.world):  # rank order, fp64
            s1 += stats[q, :, 0]
            s2 += stats[q, :, 1]
        M = np.array([key_to_float(k) for k in mk])
        zero = np.nonzero(Tt == 0)[0]
        if len(zero):
            raise AllZeroWeightError(f"all particle weights are zero at step {int(zero[0])}")
        lz = M + np.log(s1) - math.log(self.N)
        res = SmcResult(n_particles=self.N, log_z=float(lz.sum()), log_z_steps=lz, ess=s1 * s1 / s2,
                        max_log_weight=M, total_weight=Tt)
        for t, h in self.hist.items():
            hi = h.cpu().numpy().view(np.uint64).sum(axis=0)
            res.filtering_int[t] = hi
            res.filtering[t] = hi.astype(np.float64) / float(hi.sum())
        res.states = [rk.x[self.cur] for rk in self.ranks]
        res.log_weights = [self.log_weights(rk) for rk in self.ranks]
        res.ancestors = self.ancestors
        return res


def run_smc(model: HiddenMarkovModel, n_particles: int, rng, *, steps: int | None = None,
            record_ancestors: bool = False, hist_steps=None, group=None, device=None,
            local_world: int | None = None, graph: bool = False) -> SmcResult:
    """Bootstrap particle filter with systematic resampling at every step.
    graph=True captures the run as one CUDA graph (worth it when a runner is reused: see
    SmcRunner.launch)."""
    r = SmcRunner(model, n_particles, rng, group=group, device=device, record_ancestors=record_ancestors,
                  hist_steps=hist_steps, local_world=local_world, steps=steps, graph=graph)
    return r.run()
