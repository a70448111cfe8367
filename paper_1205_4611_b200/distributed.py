"""Multi-GPU evaluation: one process per GPU, subtrees partitioned across ranks.

SURVEY §8(e).  The reference is single-process (``SPEC.md:409`` lists
multi-GPU distribution as a non-goal); this module adds the domain
decomposition the north star asks for.  Rank r of G = 2^s0 ranks owns the
subtree below segment r of the first s0 median splits (a contiguous box range
on every level, a contiguous particle range); the levels above are shared and
computed redundantly.  The compute phases are libfmm2d.so kernels
(``csrc/dist.cu``); the collectives between them go through
``torch.distributed`` -- NCCL over NVLink / NVSwitch on a GPU box -- on the
same CUDA stream, so the library and the collectives are ordered without host
synchronisation except where a host needs counts (message sizes).

Collectives per evaluation (G > 1): bbox allreduce; per top split step 8
radix-select allreduces of 256 x 2^s int32 + one allgather of tie counts;
one all-to-all of the particle records; one allgather of the owned box
geometry; two halo exchanges (request ids + payload all-to-alls) for source
particles (P2P/P2L) and multipoles (M2L/M2P); one allgather of the first
owned level's multipoles.  With the ``gloo`` backend (tests: several ranks on
one device or on CPU hosts) tensors are staged through host memory.

The tree, the interaction lists and every per-target accumulation are those
of the single-GPU engine (tests compare values, lists and counts).
"""

from __future__ import annotations

import ctypes as C
import math
import time

import numpy as np

from . import _lib
from .engine import PHASE_NAMES, EngineReport, _KINDS
from .tree import ParticleSet, TreeConfig


class DeviceArray:
    """``__cuda_array_interface__`` view of library-owned device memory."""

    _TYPESTR = {"float64": "<f8", "int32": "<i4", "int64": "<i8"}

    def __init__(self, ptr: int, shape, dtype: str):
        self.__cuda_array_interface__ = {
            "shape": tuple(int(s) for s in shape), "typestr": self._TYPESTR[dtype],
            "data": (int(ptr), False), "version": 3, "strides": None}


class Comm:
    """The few collectives the distributed engine needs, on torch.distributed.

    ``nccl``: CUDA tensors in place.  Other backends (``gloo``): staged through
    host memory, so tests can run several ranks on one GPU or on CPU hosts.
    """

    def __init__(self, group=None):
        import torch.distributed as dist
        self.dist = dist
        self.group = group
        self.size = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        self.staged = dist.get_backend(group) != "nccl"
        # a one-rank group exchanges with itself only: every collective is a
        # local copy (no NCCL launch, no host round trip)
        self.solo = self.size == 1

    def _host(self, t):
        return t.cpu() if self.staged and t.is_cuda else t

    def _back(self, host, t):
        if host is not t:
            t.copy_(host)

    def allreduce(self, t, op: str = "sum"):
        ops = {"sum": self.dist.ReduceOp.SUM, "min": self.dist.ReduceOp.MIN,
               "max": self.dist.ReduceOp.MAX}
        if self.solo:
            return t
        h = self._host(t)
        self.dist.all_reduce(h, op=ops[op], group=self.group)
        self._back(h, t)
        return t

    def all_gather(self, out, inp):
        """out: ``size`` equal chunks along dim 0, rank order."""
        if self.solo:
            if out.data_ptr() != inp.data_ptr():
                out.copy_(inp.reshape(out.shape))
            return out
        hi = self._host(inp)
        if self.staged:
            chunks = [hi.new_empty(hi.shape) for _ in range(self.size)]
            self.dist.all_gather(chunks, hi.contiguous(), group=self.group)
            self._back(self._cat(chunks), out)
        else:
            self.dist.all_gather_into_tensor(out, inp.contiguous(), group=self.group)
        return out

    @staticmethod
    def _cat(chunks):
        import torch
        return torch.cat(chunks, 0)

    def all_to_all(self, out, inp, out_splits, in_splits):
        """all-to-all with row counts per peer (rank order)."""
        out_splits = [int(v) for v in out_splits]
        in_splits = [int(v) for v in in_splits]
        if self.solo:
            if out.numel():
                out.copy_(inp)
            return out
        if self.staged:
            import torch
            hi = self._host(inp)
            ho = torch.empty((sum(out_splits),) + tuple(inp.shape[1:]), dtype=inp.dtype)
            if hasattr(self.dist, "all_to_all_single") and self.dist.get_backend(self.group) != "gloo":
                self.dist.all_to_all_single(ho, hi, out_splits, in_splits, group=self.group)
            else:
                self._gloo_all_to_all(ho, hi, out_splits, in_splits)
            self._back(ho, out)
        else:
            self.dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)
        return out

    def _gloo_all_to_all(self, ho, hi, out_splits, in_splits):
        # gloo: point-to-point exchange in rank order
        ins = list(hi.split(in_splits, 0))
        outs = list(ho.split(out_splits, 0))
        ops = []
        for q in range(self.size):
            if q == self.rank:
                outs[q].copy_(ins[q])
                continue
            if in_splits[q]:
                ops.append(self.dist.P2POp(self.dist.isend, ins[q].contiguous(), q, self.group))
            if out_splits[q]:
                ops.append(self.dist.P2POp(self.dist.irecv, outs[q], q, self.group))
        if ops:
            for w in self.dist.batch_isend_irecv(ops):
                w.wait()

    def exchange_counts(self, counts):
        """counts[q] = items this rank sends to q -> items q sends to this rank."""
        import torch
        if self.solo:
            return [int(v) for v in counts]
        t = torch.tensor([int(v) for v in counts], dtype=torch.int64)
        if self.staged:
            chunks = [torch.empty_like(t) for _ in range(self.size)]
            self.dist.all_gather(chunks, t, group=self.group)
            rows = torch.stack(chunks)
        else:
            # pinned staging both ways, one stream sync (the caller needs the
            # sizes on the host anyway)
            hin, hout, g = _pinned_counts(self.size)
            hin.copy_(t)
            self.dist.all_gather_into_tensor(g, hin.to(g.device, non_blocking=True),
                                             group=self.group)
            hout.copy_(g, non_blocking=True)
            torch.cuda.current_stream(g.device).synchronize()
            rows = hout.view(self.size, self.size)
        return [int(v) for v in rows[:, self.rank]]


_streams: dict = {}
_pinned: dict = {}


def _pinned_counts(size: int):
    """(pinned send row, pinned receive matrix, device matrix) for exchange_counts."""
    import torch
    dev = torch.cuda.current_device()
    key = (dev, size)
    if key not in _pinned:
        _pinned[key] = (torch.empty(size, dtype=torch.int64).pin_memory(),
                        torch.empty(size * size, dtype=torch.int64).pin_memory(),
                        torch.empty(size * size, dtype=torch.int64,
                                    device=torch.device("cuda", dev)))
    return _pinned[key]


def engine_stream(device: int):
    """The CUDA stream a rank's library phases and collectives share."""
    import torch
    s = _streams.get(device)
    if s is None:
        s = torch.cuda.Stream(device=device)
        _streams[device] = s
    return s


def shard_bounds(n: int, size: int, rank: int) -> tuple[int, int]:
    """Contiguous input shard of `rank` (any split works: the tree depends only
    on the points; contiguous shards keep canonical order = original index)."""
    return (n * rank) // size, (n * (rank + 1)) // size


def top_split_steps(size: int) -> int:
    s0 = int(math.log2(size))
    if 1 << s0 != size:
        raise ValueError("the distributed engine needs a power-of-two number of ranks")
    return s0


def _rebuild_error(kind: str, msg: str) -> Exception:
    from .tree import DegenerateInputError
    return {"DegenerateInputError": DegenerateInputError, "ValueError": ValueError,
            "MemoryError": MemoryError}.get(kind, _lib.EngineError)(msg)


def _agreed(comm: Comm, fn):
    """Run a library phase that can fail on some ranks only -- a degenerate box
    or a median tie inside one rank's subtree, a singular shift among one rank's
    pairs -- then agree on the outcome: every rank raises the failure of the
    lowest failing rank (same exception type and message as the single-GPU
    engine), so no rank is left blocked in the next collective."""
    import torch
    if comm.solo:
        return fn()
    err = None
    try:
        out = fn()
    except (ValueError, MemoryError, _lib.EngineError) as e:   # DegenerateInputError is a ValueError
        err, out = e, None
    # one tiny MAX allreduce decides whether anyone failed; only then are the
    # messages gathered (pickled objects cost a host round trip per rank)
    flag = torch.tensor([0 if err is None else 1], dtype=torch.int32)
    if not comm.staged:
        flag = flag.cuda()
    comm.allreduce(flag, "max")
    if int(flag.item()) == 0:
        return out
    info = [None] * comm.size
    comm.dist.all_gather_object(info, None if err is None else (type(err).__name__, str(err)),
                                group=comm.group)
    for q, e in enumerate(info):
        if e is not None:
            if q == comm.rank:
                raise err
            raise _rebuild_error(*e)
    return out


def evaluate_shard(ctx: _lib.Context, comm: Comm, n_total: int, d_pos, d_gamma, index_base: int,
                   cfg: TreeConfig, evals=None):
    """One rank's part of a distributed evaluation.

    ``d_pos`` (float64 [n_local, 2]) / ``d_gamma`` (float64 [n_local]) are this
    rank's shard of the sources on its GPU, original indices starting at
    ``index_base`` (shards of consecutive ranks must be consecutive).
    ``evals`` = (m_total, d_epos float64 [m_local, 2], eval_index_base) for
    separate evaluation points, sharded the same way (None: the evaluation
    points alias the sources).  Returns (values complex as float64 [n_own, 2]
    in tree order, their original evaluation indices int64 [n_own], library
    Report of this rank).
    """
    import torch
    lib, h = ctx.lib, ctx.h
    G, rank = comm.size, comm.rank
    s0 = top_split_steps(G)
    dev = d_pos.device
    f64, i32, i64 = torch.float64, torch.int32, torch.int64
    stream = torch.cuda.current_stream(dev).cuda_stream
    if not stream:
        raise ValueError("run evaluate_shard under a non-default torch.cuda.Stream (the library "
                         "and the collectives share it)")
    nlev = C.c_int32()
    ctx.check(lib.fmm2d_dist_setup(h, G, rank, int(n_total), int(cfg.p_terms), float(cfg.theta),
                                   int(cfg.n_desired_per_box), C.c_void_p(stream),
                                   C.byref(nlev)))
    L = int(nlev.value)
    n_local = int(d_pos.shape[0])
    bbox = torch.empty(4, dtype=f64, device=dev)
    ctx.check(lib.fmm2d_dist_load(h, n_local, C.c_void_p(d_pos.data_ptr()),
                                  C.c_void_p(d_gamma.data_ptr()), int(index_base),
                                  C.c_void_p(bbox.data_ptr())))
    if evals is not None:
        m_total, d_epos, e_base = evals
        ctx.check(lib.fmm2d_dist_load_evals(h, int(m_total), int(d_epos.shape[0]),
                                            C.c_void_p(d_epos.data_ptr()), int(e_base),
                                            C.c_void_p(bbox.data_ptr())))
    comm.allreduce(bbox, "min")
    ctx.check(lib.fmm2d_dist_root(h, C.c_void_p(bbox.data_ptr())))
    # top split: s0 exact median steps, collectively
    for s in range(s0):
        nseg = 1 << s
        if s % 2 == 0 and s > 0 and s // 2 < L:
            box = torch.empty(4 * nseg, dtype=f64, device=dev)
            ctx.check(lib.fmm2d_dist_segbox(h, s, C.c_void_p(box.data_ptr())))
            comm.allreduce(box, "min")
            ctx.check(lib.fmm2d_dist_check_segbox(h, s, C.c_void_p(box.data_ptr())))
        hist = torch.empty(256 * nseg, dtype=i32, device=dev)
        for rho in range(8):
            ctx.check(lib.fmm2d_dist_hist(h, s, rho, C.c_void_p(hist.data_ptr())))
            comm.allreduce(hist, "sum")
            ctx.check(lib.fmm2d_dist_pick(h, s, rho, C.c_void_p(hist.data_ptr())))
        eq = torch.empty(nseg, dtype=i32, device=dev)
        ctx.check(lib.fmm2d_dist_eqcount(h, s, C.c_void_p(eq.data_ptr())))
        eq_all = torch.empty(G * nseg, dtype=i32, device=dev)
        comm.all_gather(eq_all, eq)
        ctx.check(lib.fmm2d_dist_partition(h, s, C.c_void_p(eq_all.data_ptr())))
    # records to their subtree's rank
    counts = np.zeros(G, np.int64)
    rec_ptr = C.c_void_p()
    ctx.check(lib.fmm2d_dist_send_counts(h, _lib.iptr(counts), C.byref(rec_ptr)))
    send = torch.as_tensor(DeviceArray(rec_ptr.value or 0, (n_local, 4), "float64"), device=dev) \
        if n_local else torch.empty((0, 4), dtype=f64, device=dev)
    recv_counts = comm.exchange_counts(counts)
    recv = torch.empty((sum(recv_counts), 4), dtype=f64, device=dev)
    comm.all_to_all(recv, send, recv_counts, counts)
    erecv = None
    if evals is not None:
        # evaluation points to the rank owning their top-split segment (coord <= cut)
        ecounts = np.zeros(G, np.int64)
        eptr = C.c_void_p()
        ctx.check(lib.fmm2d_dist_eval_route(h, _lib.iptr(ecounts), C.byref(eptr)))
        m_loc = int(ecounts.sum())
        esend = (torch.as_tensor(DeviceArray(eptr.value or 0, (m_loc, 4), "float64"), device=dev)
                 if m_loc else torch.empty((0, 4), dtype=f64, device=dev))
        erecv_counts = comm.exchange_counts(ecounts)
        erecv = torch.empty((sum(erecv_counts), 4), dtype=f64, device=dev)
        comm.all_to_all(erecv, esend, erecv_counts, ecounts)
    own = np.zeros(1, np.int64)
    e_ptr = C.c_void_p(erecv.data_ptr()) if erecv is not None and erecv.shape[0] else None
    m_recv = 0 if erecv is None else erecv.shape[0]
    _agreed(comm, lambda: ctx.check(lib.fmm2d_dist_build(h, C.c_void_p(recv.data_ptr()),
                                                         recv.shape[0], e_ptr, m_recv,
                                                         _lib.iptr(own))))
    geo = torch.empty(int(own[0]) * 5, dtype=f64, device=dev)
    ctx.check(lib.fmm2d_dist_geom_pack(h, C.c_void_p(geo.data_ptr())))
    geo_all = torch.empty(G * int(own[0]) * 5, dtype=f64, device=dev)
    comm.all_gather(geo_all, geo)
    req = np.zeros(2 * G, np.int64)
    _agreed(comm, lambda: ctx.check(lib.fmm2d_dist_connect(h, C.c_void_p(geo_all.data_ptr()),
                                                           _lib.iptr(req))))

    def exchange(kind):
        mine = [int(v) for v in req[kind * G:(kind + 1) * G]]
        theirs = comm.exchange_counts(mine)
        ptr = C.c_void_p()
        ctx.check(lib.fmm2d_dist_requests(h, kind, C.byref(ptr)))
        n_mine = sum(mine)
        my_ids = (torch.as_tensor(DeviceArray(ptr.value, (n_mine,), "int32"), device=dev)
                  if n_mine else torch.empty(0, dtype=i32, device=dev))
        ids_in = torch.empty(sum(theirs), dtype=i32, device=dev)
        comm.all_to_all(ids_in, my_ids, theirs, mine)
        item = np.zeros(1, np.int64)
        ctx.check(lib.fmm2d_dist_item_doubles(h, kind, _lib.iptr(item)))
        payload = torch.empty((ids_in.shape[0], int(item[0])), dtype=f64, device=dev)
        ctx.check(lib.fmm2d_dist_pack(h, kind, C.c_void_p(ids_in.data_ptr()), ids_in.shape[0],
                                      C.c_void_p(payload.data_ptr())))
        answers = torch.empty((n_mine, int(item[0])), dtype=f64, device=dev)
        comm.all_to_all(answers, payload, mine, theirs)
        ctx.check(lib.fmm2d_dist_unpack(h, kind, C.c_void_p(answers.data_ptr())))
        return answers                                  # keep alive until the stream consumed it

    keep = [exchange(1)]                                 # halo particles (P2P, P2L)
    lt = (s0 + 1) // 2
    cnt = 1 << (2 * lt - s0)
    row = 2 * (int(cfg.p_terms) + 1)
    top = torch.empty(cnt * row, dtype=f64, device=dev)
    nb = np.zeros(1, np.int64)
    ctx.check(lib.fmm2d_dist_upward(h, C.c_void_p(top.data_ptr()), _lib.iptr(nb)))
    top_all = torch.empty(G * cnt * row, dtype=f64, device=dev)
    comm.all_gather(top_all, top)
    ctx.check(lib.fmm2d_dist_upward_top(h, C.c_void_p(top_all.data_ptr())))
    keep.append(exchange(0))                             # halo multipoles (M2L, M2P)
    n_own = recv.shape[0] if erecv is None else erecv.shape[0]
    vals = torch.empty((n_own, 2), dtype=f64, device=dev)
    idx = torch.empty(n_own, dtype=i64, device=dev)
    rep = _lib.Report()
    _agreed(comm, lambda: ctx.check(lib.fmm2d_dist_downward(
        h, C.c_void_p(vals.data_ptr()), C.c_void_p(idx.data_ptr()), C.byref(rep))))
    return vals, idx, rep


def _merge_report(ctx, comm: Comm, rep: _lib.Report, wall: float, m: int) -> EngineReport:
    import torch
    ph = torch.tensor(list(rep.phase_ms)[:8] + [rep.device_ms], dtype=torch.float64)
    cnt = torch.tensor([rep.p2p_skips] + list(rep.list_totals), dtype=torch.int64)
    if not comm.staged:
        ph, cnt = ph.cuda(), cnt.cuda()
    comm.allreduce(ph, "max")
    comm.allreduce(cnt, "sum")
    ph, cnt = ph.cpu().tolist(), cnt.cpu().tolist()
    hist = {}
    for k, name in enumerate(_KINDS):
        nb = int(rep.max_len[k]) + 1
        hh = np.zeros(nb, np.int64)
        ctx.check(ctx.lib.fmm2d_histogram(ctx.h, k, _lib.iptr(hh), nb))
        hist[name] = {int(i): int(c) for i, c in enumerate(hh) if c}
    parts = [None] * comm.size
    comm.dist.all_gather_object(parts, hist, group=comm.group)
    merged = {name: {} for name in _KINDS}
    for part in parts:
        for name, hd in part.items():
            for k, v in hd.items():
                merged[name][k] = merged[name].get(k, 0) + v
    phases = {name: ph[i] * 1e-3 for i, name in enumerate(PHASE_NAMES[:-1])}
    phases["other"] = max(0.0, wall - sum(phases.values()))
    return EngineReport(
        phase_seconds=phases, total_seconds=wall, n_levels=int(rep.n_levels),
        n_boxes=int(rep.n_boxes), finest_src_min=int(rep.finest_src_min),
        finest_src_max=int(rep.finest_src_max), finest_src_mean=float(rep.finest_src_mean),
        list_histograms={k: dict(sorted(v.items())) for k, v in merged.items()},
        coincident_skips=max(0, int(cnt[0]) - m), parallel=False,
        device_seconds=ph[8] * 1e-3,
        list_totals={name: int(cnt[1 + k]) for k, name in enumerate(_KINDS)},
        kernel_launches=int(rep.kernel_launches))


def fmm_evaluate_distributed(points: ParticleSet, cfg: TreeConfig | None = None, *, group=None,
                             device: int | None = None, gather: bool = True):
    """SPMD drop-in for ``fmm_evaluate`` (engine.py:207-279) across the ranks of
    ``group`` (one GPU each): every rank passes the same point set, uploads its
    shard of the sources (and of separate evaluation points), and
    (``gather=True``) receives all values in input order.

    ``gather=False`` returns ``(values_owned complex128, original_indices)`` of
    the evaluation points this rank owns instead of the full array.

    Aliased evaluation points follow the sources' median splits; when a
    coordinate tie straddles a cut the reference's evaluation split (coord <=
    cut, tree.py:205-215) differs from the source split, and -- like the
    single-GPU engine -- the evaluation reruns with the points handled as
    separate evaluation points (every rank reruns together: the tie is agreed).
    """
    import torch
    t0 = time.perf_counter()
    cfg = cfg or TreeConfig()
    comm = Comm(group)
    dev_index = torch.cuda.current_device() if device is None else int(device)
    dev = torch.device("cuda", dev_index)
    ctx = _lib.default_context(dev_index)
    n, m = points.n_sources, points.n_evals
    lo, hi = shard_bounds(n, comm.size, comm.rank)
    separate = not points.evals_alias_sources
    with ctx.lock, torch.cuda.device(dev), torch.cuda.stream(engine_stream(dev_index)):
        pos = torch.from_numpy(np.ascontiguousarray(points.positions[lo:hi])
                               .view(np.float64).reshape(-1, 2)).to(dev)
        gam = torch.from_numpy(np.ascontiguousarray(points.strengths[lo:hi])).to(dev)

        def run(as_separate):
            evals = None
            if as_separate:
                elo, ehi = shard_bounds(m, comm.size, comm.rank)
                src = points.eval_positions if separate else points.positions
                epos = torch.from_numpy(np.ascontiguousarray(src[elo:ehi])
                                        .view(np.float64).reshape(-1, 2)).to(dev)
                evals = (m, epos, elo)
            return evaluate_shard(ctx, comm, n, pos, gam, lo, cfg, evals)

        # the library stays on the engine stream (dist_end) until the gather's
        # scatter kernel and the report queries are done
        try:
            try:
                vals, idx, rep = run(separate)
            except ValueError as e:
                if separate or "ties" not in str(e):
                    raise
                vals, idx, rep = run(True)
            return _gather_and_report(ctx, comm, dev, vals, idx, rep, gather, m,
                                      0 if separate else n, t0)
        finally:
            ctx.lib.fmm2d_dist_end(ctx.h)


def _gather_and_report(ctx, comm, dev, vals, idx, rep, gather, m, self_skips, t0):
    """Values of all evaluation points in input order (gather) or this rank's
    owned ones, plus the merged report; runs on the engine stream."""
    import torch
    if gather:
        n_max = torch.tensor([vals.shape[0]], dtype=torch.int64)
        if not comm.staged:
            n_max = n_max.to(dev)
        comm.allreduce(n_max, "max")
        nm = int(n_max.item())
        pv = torch.zeros((nm, 2), dtype=torch.float64, device=dev)
        pi = torch.full((nm,), -1, dtype=torch.int64, device=dev)
        pv[:vals.shape[0]] = vals
        pi[:idx.shape[0]] = idx
        av = torch.empty((comm.size * nm, 2), dtype=torch.float64, device=dev)
        ai = torch.empty(comm.size * nm, dtype=torch.int64, device=dev)
        comm.all_gather(av, pv)
        comm.all_gather(ai, pi)
        keep = ai >= 0
        av, ai = av[keep].contiguous(), ai[keep].contiguous()
        out = torch.empty((m, 2), dtype=torch.float64, device=dev)
        ctx.check(ctx.lib.fmm2d_scatter_values(ctx.h, ai.shape[0], C.c_void_p(av.data_ptr()),
                                               C.c_void_p(ai.data_ptr()),
                                               C.c_void_p(out.data_ptr())))
        values = out.cpu().numpy().view(np.complex128).reshape(-1)
    else:
        values = (vals.cpu().numpy().view(np.complex128).reshape(-1), idx.cpu().numpy())
    torch.cuda.current_stream(dev).synchronize()
    wall = time.perf_counter() - t0
    # coincident_skips excludes the points' meetings with themselves only
    # when the evaluation points alias the sources (engine.py:271-275)
    report = _merge_report(ctx, comm, rep, wall, self_skips)
    report.total_seconds = time.perf_counter() - t0
    return values, report
