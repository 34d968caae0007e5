"""Multi-GPU merge: row-block sharding of Q_old with index-sharded roots.

One process per GPU (torch.distributed, NCCL over NVLink/NVSwitch).  For one merge:

* roots, Loewner weights and column normalizers are sharded by index
  (rank r owns [r*c, (r+1)*c), c = ceil(k / world)); lam/gamma/mu, zhat and v are
  all-gathered (3k + 2k doubles);
* the sample products are sharded by rows: rank r computes rows of Y = C Omega and of
  Z = C^T Omega in its index range; Y and Z are all-gathered (2 k ws doubles);
* partition, rank estimate, the sample draw and the HSS construction are replicated
  (every rank holds the whole tree: D and B are regenerated from the generators,
  never sent);
* the multiply Q_new = Q_old H is row-local: Q_old never moves.

The driver is written against a small ``ops`` interface so the same sharding /
gathering logic runs on the GPU (``GpuOps``: libhsseig_b200.so through the C ABI) and,
in the CPU test-suite, with gloo and a NumPy stand-in.
"""
import ctypes

import numpy as np
import torch
import torch.distributed as dist

from .flops import cauchy_eval_flops, gemm_flops, secular_flops
from .hss import build_partition, rank_bound
from .secular import SecularConvergenceError, WeightRecomputationError


def shard_range(k, rank, world):
    """Index shard [lo, hi) of rank in a padded even split (chunk = ceil(k / world))."""
    c = -(-k // world)
    lo = min(k, rank * c)
    return lo, min(k, lo + c), c


def _all_gather(parts, t, group=None):
    """dist.all_gather; CUDA tensors go through host memory on a gloo group (the CPU test
    backend), NCCL gathers them in place."""
    if t.is_cuda and dist.get_backend(group) == "gloo":
        hp = [torch.empty(p.shape, dtype=p.dtype) for p in parts]
        dist.all_gather(hp, t.cpu(), group=group)
        for p, h in zip(parts, hp):
            p.copy_(h)
        return
    dist.all_gather(parts, t, group=group)


def gather_rows(local, chunk, k, group=None):
    """All-gather equal-size row chunks (padded to `chunk` rows) and trim to k rows."""
    world = dist.get_world_size(group)
    if local.shape[0] < chunk:
        pad = torch.zeros((chunk - local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
        local = torch.cat([local, pad])
    parts = [torch.empty_like(local) for _ in range(world)]
    _all_gather(parts, local.contiguous(), group)
    return torch.cat(parts)[:k]


class PeerBuffers:
    """Full-size float64 buffers that every rank of `group` stores into directly: each rank
    allocates its own, shares them through CUDA IPC (torch's own handle export) and maps the
    others', so a kernel can write its block of a result into all ranks' copies over
    NVLink / NVSwitch (one process per GPU; on one device across processes in the tests).
    `ptrs[b]` is the device array of the ranks' base pointers of buffer b (rank order)."""

    def __init__(self, shapes, group=None):
        from torch.multiprocessing.reductions import reduce_tensor
        self.local = [torch.zeros(sh, dtype=torch.float64, device="cuda") for sh in shapes]
        torch.cuda.synchronize()
        world = dist.get_world_size(group)
        rank = dist.get_rank(group)
        me = torch.cuda.current_device()
        self.views, self.ptrs = [], []
        # every step below is agreed on by the whole group, so a rank that cannot export or
        # map a peer buffer makes all ranks fall back to the NCCL gather together
        try:
            mine = (me, [reduce_tensor(t) for t in self.local])
        except Exception:          # noqa: BLE001 (no CUDA IPC here)
            mine = None
        handles = [None] * world
        dist.all_gather_object(handles, mine, group=group)
        ok = all(h is not None for h in handles) and all(
            dv == me or torch.cuda.can_device_access_peer(me, dv) for dv, _ in handles)
        if ok:
            try:
                for b in range(len(shapes)):
                    ts = []
                    for r in range(world):
                        if r == rank:
                            ts.append(self.local[b])
                        else:
                            fn, args = handles[r][1][b]
                            ts.append(fn(*args))
                    self.views.append(ts)          # keeps the peers' mappings alive
                    self.ptrs.append(torch.tensor([t.data_ptr() for t in ts], dtype=torch.int64,
                                                  device="cuda"))
            except Exception:      # noqa: BLE001 (a peer mapping failed)
                ok = False
        oks = [None] * world
        dist.all_gather_object(oks, ok, group=group)
        self.ok = all(oks)                 # one decision for the whole group
        self.group = group
        if not self.ok:
            self.views, self.ptrs = [], []

    def close(self):
        """Unmap the peers' buffers before anyone frees its own: every rank drains its
        stream, the group agrees, the imported views are dropped, and the group agrees again
        (an exporter that exits while an importer still maps its memory can take the
        importer down at teardown)."""
        if not self.views and not self.local:
            return
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        self.views, self.ptrs = [], []
        import gc
        gc.collect()
        torch.cuda.synchronize()
        dist.barrier(group=self.group)
        self.local = []


_FENCE = {}


def peer_fence(group=None):
    """Every rank's peer stores so far have landed before this rank's stream goes on.

    NCCL: a one-element all-reduce enqueued on the compute stream is the fence, with no host
    drain.  It completes on a rank only once every rank's stream has reached it, i.e. after
    every rank's peer-store kernels retired (they end with a system-scope fence), and the
    work enqueued after it on this rank's stream waits for it.  The alternating buffer sets
    of GpuOps.sample_gather rely on the same ordering (a rank overwrites set n % 2 only
    after fence n - 1, which every rank reaches after its reads of set n - 2).
    Other backends (gloo ranks sharing one device in the tests): the stream is drained on
    the host and the group barriers."""
    if dist.get_backend(group) == "nccl":
        dev = torch.cuda.current_device()
        t = _FENCE.get(dev)
        if t is None:
            t = _FENCE[dev] = torch.zeros(1, dtype=torch.int32, device="cuda")
        dist.all_reduce(t, group=group)
        return
    torch.cuda.current_stream().synchronize()
    dist.barrier(group=group)


def _host_copy(ts):
    """Small device tensors to pinned host memory behind the current stream (async, one
    event); CPU tensors (the gloo test ops) are taken as they are."""
    if not ts[0].is_cuda:
        return [t.clone() for t in ts], None
    hs = [torch.empty(t.shape, dtype=t.dtype, pin_memory=True) for t in ts]
    for h, t in zip(hs, ts):
        h.copy_(t, non_blocking=True)
    ev = torch.cuda.Event()
    ev.record()
    return hs, ev


def _host_wait(p):
    hs, ev = p
    if ev is not None:
        ev.synchronize()
    return [h.numpy() for h in hs]


def rank_from(part, span, mu_h, eps, cap):
    """estimate_rank (hss.py:87-103) from host copies of the boundary gaps."""
    if part.n_leaves < 2:
        return 0
    r = 0
    for lo, _ in part.ranges[1:]:
        r = max(r, rank_bound(max(span / mu_h[lo - 1], 1.0), eps))
    return min(max(r, 1), cap)


class ShardedMerge:
    """One merge over the ranks of `group`; each rank holds rows of Q_old."""

    def __init__(self, k, cfg, ops, group=None):
        self.k, self.cfg, self.ops, self.group = int(k), cfg, ops, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)

    def run(self, d, z, rho, X, seed, rows_total=None):
        """rows_total: rows of the whole Q block over all ranks (the merge order in a full
        solve) for the record's flop counts; summed over the group when not given."""
        k, cfg, ops = self.k, self.cfg, self.ops
        lo, hi, c = shard_range(k, self.rank, self.world)
        info = {"used_hss": False, "fell_back": False, "r_used": 0}
        marks = []   # (phase that ends here, CUDA event) on the compute stream: bench phases

        def mark(name):
            if X.is_cuda:
                e = torch.cuda.Event(enable_timing=True)
                e.record()
                marks.append((name, e))

        mark("start")
        if rows_total is None:
            cnt = gather_rows(torch.tensor([[float(X.shape[0])]], dtype=torch.float64,
                                           device=X.device), 1, self.world, self.group)
            rows_total = int(cnt.sum())
        # roots of this rank's index shard, then the full arrays on every rank
        lam_l, gam_l, mu_l, st_l = ops.secular_part(d, z, rho, lo, hi)
        full = gather_rows(torch.stack([lam_l, gam_l, mu_l], 1), c, k, self.group)
        lam, gam, mu = full[:, 0].contiguous(), full[:, 1].contiguous(), full[:, 2].contiguous()
        st = gather_rows(st_l.view(1, -1), 1, self.world, self.group)   # world x 3
        # what the host decides on (bracket status, the pole gaps for the partition, the
        # span) comes back through async pinned copies while Loewner / normalizers run
        pend = _host_copy([st.reshape(-1).to(torch.int64),
                           torch.cat([mu.reshape(-1), torch.stack([d[0], d[-1], gam[-1]])])])
        mark("secular")
        dn = ops.dnext(d, gam, mu)
        zh_l, rad_l = ops.loewner_part(d, dn, gam, mu, z, rho, lo, hi)
        zh = gather_rows(zh_l, c, k, self.group).contiguous()
        rad = gather_rows(rad_l.view(1, -1), 1, self.world, self.group)
        pend_rad = _host_copy([rad.reshape(-1).to(torch.int64)])
        v_l = ops.normalizers_part(d, dn, gam, mu, zh, lo, hi)
        v = gather_rows(v_l, c, k, self.group).contiguous()
        st_h, muh = _host_wait(pend)
        st_h = st_h.reshape(self.world, -1)
        iters = int(st_h[:, 0].sum())
        bad_g = int(st_h[:, 1].min())
        bad_m = int(st_h[:, 2].min())
        bad = bad_g if bad_g < k else (bad_m if (k >= 2 and bad_m < k) else -1)
        if bad >= 0:
            raise SecularConvergenceError(f"root {bad} lost its bracket")
        mu_h, (d0_h, dl_h, gl_h) = muh[:k], muh[k:]

        def check_weights():
            rmin = int(_host_wait(pend_rad)[0].min())
            if rmin < k:
                raise WeightRecomputationError(f"non-positive radicand at index {rmin}")

        info["iterations"] = iters
        info["flops_secular"] = secular_flops(k, iters) + 14 * k * k
        mark("loewner_normalizers")
        gen = ops.generators(d, dn, gam, mu, zh, v)
        tree = None
        if cfg.method == "adc-srrsc" and k > cfg.hss_threshold:
            # ADC1: no sample; the construction is partitioned by subtree like ADC2's
            try:
                part = build_partition(k, cfg.leaf_size, None, None, mu_h)
            except ValueError:
                part = None
            if part is not None:
                cap = min(part.min_leaf, ops.max_width)
                tree = ops.build_srrsc(gen, part, cap, cfg.srrsc_tol, self.group)
                mark("build")
        elif cfg.method == "adc-rand" and k > cfg.hss_threshold:
            try:
                part = build_partition(k, cfg.leaf_size, None, None, mu_h)
            except ValueError:
                part = None
            if part is not None:
                span = float((dl_h + gl_h) - d0_h)
                r = min(rank_from(part, span, mu_h, cfg.rank_eps, cfg.rank_cap),
                        part.min_leaf - cfg.oversample)
                w = r + cfg.oversample
                if r >= 1 and w <= ops.max_width:
                    om = ops.omega(seed, k, w)
                    mark("partition_omega")
                    # the off-diagonal sample (default) masks the leaves' diagonal blocks
                    offdiag = getattr(cfg, "sample", "offdiag") == "offdiag"
                    mask = part if offdiag else None
                    fused = getattr(ops, "sample_gather", None)
                    YZ = fused(gen, om, w, lo, hi, self.group, mask) if fused else None
                    if YZ is not None:
                        # sample rows stored straight into every rank's Y / Z (one kernel
                        # for the split-K reduction and the all-gather), then one fence
                        Y, Z = YZ
                        info["sample_gather"] = "peer"
                    else:
                        info["sample_gather"] = "nccl"
                        Y_l, Z_l = ops.sample_part(gen, om, w, lo, hi, mask)
                        Y = gather_rows(Y_l, c, k, self.group)
                        Z = gather_rows(Z_l, c, k, self.group)
                    mark("sample_gather")
                    tree = ops.build(gen, part, w, om, Y, Z, self.group, offdiag)
                    mark("build")
        check_weights()   # the construction has synchronised: the radicands are long back
        if tree is not None and not ops.flagged(tree):
            info["used_hss"] = True
            info["r_used"] = ops.r_used(tree)
            timed = X.is_cuda
            if timed:   # the row-local multiply's device time (bench's roofline)
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
            out = ops.multiply(X, tree)
            if timed:
                e1.record()
                info["multiply_events"] = (e0, e1)
                marks.append(("multiply", e1))
        else:
            out = ops.dense(X, gen)
            mark("dense")
        # the reference notes a fallback whenever the HSS route was taken and the dense
        # product ran instead: no partition, r < 1, a flagged tree (dc.py:147-160); here
        # also a sample wider than the kernels' MAX_WIDTH
        eligible = cfg.method in ("adc-rand", "adc-srrsc") and k > cfg.hss_threshold
        info["fell_back"] = bool(eligible and not info["used_hss"])
        # per-phase counts under the reference's conventions (flops.py), all rows_total rows
        fl = {"secular": info["flops_secular"], "update_dense": 0, "hss_construct": 0,
              "hss_mult": 0}
        if tree is not None:
            fl["hss_construct"] = ops.construct_flops(tree)
        if info["used_hss"]:
            fl["hss_mult"] = ops.mult_flops(tree, rows_total)
        else:
            fl["update_dense"] = cauchy_eval_flops(k * k) + gemm_flops(rows_total, k, k)
        info["flops"] = fl
        info["rows_total"] = rows_total
        info["tree"] = tree
        info["marks"] = marks
        return lam, out, info


def subtree_layout(depth, s_lev):
    """Postorder node-id ranges and leaf ranges of the 2^s_lev subtrees rooted at level s_lev."""
    size = (1 << (depth - s_lev + 1)) - 1
    blocks, leaves = [], []

    def rec(level, pos, first):
        # first = postorder id of the first node of the subtree rooted at (level, pos)
        if level == s_lev:
            blocks.append((first, first + size))
            nl = 1 << (depth - s_lev)
            leaves.append((pos * nl, (pos + 1) * nl))
            return first + size
        nxt = rec(level + 1, 2 * pos, first)
        nxt = rec(level + 1, 2 * pos + 1, nxt)
        return nxt + 1

    rec(0, 0, 0)
    return blocks, leaves


def gather_subtrees(tree, s_lev, group=None):
    """All-gather what the other ranks built for their subtrees, in one collective: every
    node's ranks, flags, skeletons, U, V^T and B (what the multiply and the upper levels
    read), the leaves' D, and only for the subtree roots the selected rows and
    compressions the upper levels consume."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    ct = tree.ct
    depth, ws, pmax, dld = ct.depth, ct.ws, ct.pmax, ct.dld
    blocks, leaves = subtree_layout(depth, s_lev)
    roots = [(b - 1, b) for _, b in blocks]          # a subtree root is last in its block
    per_node = {"rU": 4, "rV": 4, "flags": 8, "rres": 8, "cres": 8, "rsel": 4 * ws, "csel": 4 * ws,
                "rloc": 4 * ws, "cloc": 4 * ws, "U": 8 * pmax * ws, "Vt": 8 * ws * pmax,
                "B": 8 * ws * ws}
    root_only = {"psel": 8 * ws * ws, "tsel": 8 * ws * ws, "ycomp": 8 * ws * ws,
                 "zcomp": 8 * ws * ws}
    base = tree.mem.data_ptr()
    drows = (ct.mmax + 1 + 15) // 16 * 16 + 2
    regions = ([(name, nb, blocks) for name, nb in per_node.items()]
               + [(name, nb, roots) for name, nb in root_only.items()]
               + [("D", 8 * drows * dld, leaves)])
    spans = []
    for name, nb, rng in regions:
        off = getattr(ct, name) - base
        spans.append([(off + a * nb, off + b * nb) for a, b in rng])
    mine = torch.cat([tree.mem[sp[rank][0]:sp[rank][1]] for sp in spans])
    parts = [torch.empty_like(mine) for _ in range(world)]
    _all_gather(parts, mine, group)
    for r in range(world):
        if r == rank:
            continue
        pos = 0
        for sp in spans:
            a, b = sp[r]
            tree.mem[a:b].copy_(parts[r][pos:pos + (b - a)])
            pos += b - a


class GpuOps:
    """Device implementation of the ShardedMerge ops through libhsseig_b200.so."""

    def __init__(self, k):
        from . import _native as nat
        from . import sample_rng
        from .hss import MAX_WIDTH
        self.nat, self.lib, self.k = nat, nat.load(), int(k)
        self.max_width = MAX_WIDTH
        f64 = dict(dtype=torch.float64, device="cuda")
        self.swork = torch.empty(2 * self.k + 64, **f64)
        self.status = torch.zeros(8, dtype=torch.int64, device="cuda")
        self._sample_k = self.k
        self.sample_work = torch.empty(int(self.lib.hsseig_sample_work_doubles(self.k, MAX_WIDTH)), **f64)
        self.rng = sample_rng.NormalStream(self.k * MAX_WIDTH) if sample_rng.available() else None
        self._trees = {}
        self._mwork = None
        self._swork = None
        self._peer = None
        self._peer_key = None
        self._peer_n = 0

    def _s(self):
        return self.nat.stream_ptr()

    def close(self):
        """Release the CUDA-IPC peer buffers in group order (call on every rank before
        destroy_process_group)."""
        for pb in self._peer or []:
            pb.close()
        self._peer, self._peer_key = None, None

    def _fit(self, k):
        # the ops serve merges of any order up to the one they were sized for
        if 2 * k + 64 > self.swork.numel():
            self.swork = torch.empty(2 * k + 64, dtype=torch.float64, device="cuda")
        if k > self._sample_k:
            from .hss import MAX_WIDTH
            self.sample_work = None
            self.sample_work = torch.empty(int(self.lib.hsseig_sample_work_doubles(k, MAX_WIDTH)),
                                           dtype=torch.float64, device="cuda")
            self._sample_k = k

    def secular_part(self, d, z, rho, lo, hi):
        nat, n = self.nat, hi - lo
        self.k = int(d.numel())
        self._fit(self.k)
        lam = torch.empty(n, dtype=torch.float64, device="cuda")
        gam, mu = torch.empty_like(lam), torch.empty_like(lam)
        its = torch.empty(n, dtype=torch.int32, device="cuda")
        self.status.zero_()
        self.status[1:4] = self.k
        nat.check(self.lib.hsseig_secular_part(nat.ptr(d), nat.ptr(z), self.k, float(rho), lo, hi,
                                               nat.ptr(lam), nat.ptr(gam), nat.ptr(mu), nat.ptr(its),
                                               nat.ptr(self.swork), nat.ptr(self.status), self._s()),
                  "secular_part")
        return lam, gam, mu, self.status[:3].clone()

    def dnext(self, d, gam, mu):
        nat = self.nat
        dn = torch.empty_like(d)
        nat.check(self.lib.hsseig_dnext(nat.ptr(d), nat.ptr(gam), nat.ptr(mu), self.k, nat.ptr(dn),
                                        self._s()), "dnext")
        return dn

    def loewner_part(self, d, dn, gam, mu, z, rho, lo, hi):
        nat = self.nat
        zh = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        self.status[3] = self.k
        nat.check(self.lib.hsseig_loewner_part(nat.ptr(d), nat.ptr(dn), nat.ptr(gam), nat.ptr(mu),
                                               nat.ptr(z), self.k, float(rho), lo, hi, nat.ptr(zh),
                                               nat.ptr(self.status), self._s()), "loewner_part")
        return zh, self.status[3:4].clone()

    def normalizers_part(self, d, dn, gam, mu, zh, lo, hi):
        nat = self.nat
        v = torch.empty(hi - lo, dtype=torch.float64, device="cuda")
        nat.check(self.lib.hsseig_normalizers_part(nat.ptr(d), nat.ptr(dn), nat.ptr(gam), nat.ptr(mu),
                                                   nat.ptr(zh), self.k, lo, hi, nat.ptr(v),
                                                   self._s()), "normalizers_part")
        return v

    def generators(self, d, dn, gam, mu, zh, v):
        from .cauchy import CauchyEvecMatrix
        return CauchyEvecMatrix(d, gam, mu, zh, v, dnext=dn)

    def omega(self, seed, k, w):
        ws = (w + 15) // 16 * 16
        om = torch.zeros(k, ws, dtype=torch.float64, device="cuda")
        if self.rng is not None:
            if k * w > self.rng.nmax:
                from . import sample_rng
                self.rng = sample_rng.NormalStream(k * w)
            flat = torch.empty(k * w, dtype=torch.float64, device="cuda")
            self.rng.draw(seed, k * w, flat)
            self.rng.fixup()
            om[:, :w] = flat.view(k, w)
        else:
            om[:, :w] = torch.as_tensor(np.random.default_rng(seed).standard_normal((k, w)),
                                        device="cuda")
        return om

    def tree_for(self, part, w):
        """The construction's tree (cached per partition and width); its leaf_of masks the
        off-diagonal sample."""
        from .hss import HssTree
        key = (part.ranges, w)
        if key not in self._trees:
            self._trees = {key: HssTree(part, w)}
        return self._trees[key]

    def _leaf_of(self, part, w):
        return self.tree_for(part, w).ct.leaf_of if part is not None else None

    def sample_part(self, gen, om, w, lo, hi, part=None):
        """Rows [lo, hi) of Y = C Omega and Z = C^T Omega; with `part` the off-diagonal
        sample (the partition's diagonal leaf blocks masked)."""
        nat = self.nat
        ws = om.shape[1]
        Y = torch.empty(hi - lo, ws, dtype=torch.float64, device="cuda")
        Z = torch.empty_like(Y)
        nat.check(self.lib.hsseig_cauchy_sample_part(gen.gen, self._leaf_of(part, w), nat.ptr(om),
                                                     ws, w, lo, hi, nat.ptr(Y), nat.ptr(Z), ws,
                                                     nat.ptr(self.sample_work), self._s()),
                  "cauchy_sample_part")
        return Y, Z

    def sample_gather(self, gen, om, w, lo, hi, group=None, part=None):
        """Y = C Omega, Z = C^T Omega on every rank with this rank's rows [lo, hi) computed
        here and stored into all ranks' copies by the reduction kernels (CUDA IPC peers);
        None when the fused path does not apply (one rank, HSSEIG_PEER=0, a panel above the
        materialisation cap), and the caller all-gathers through NCCL instead."""
        import os
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        if world < 2 or os.environ.get("HSSEIG_PEER", "1") == "0":
            return None
        nat = self.nat
        k, ws = self.k, om.shape[1]
        # one decision for the whole group, taken before anything is launched: every rank
        # tests the padded shard size c they all share (a shorter last shard fits whenever
        # c does), so no rank can take the peer path while another all-gathers
        c = -(-k // world)
        if not self.lib.hsseig_sample_peers_fits(k, c, w):
            return None
        key = (k, ws, id(group))
        if self._peer_key != key:
            # two sets, alternating: a rank writes set n % 2 only after every rank passed
            # the fence of call n - 1, i.e. finished reading set (n - 1) % 2 ... n - 2
            self._peer = [PeerBuffers([(k, ws), (k, ws)], group) for _ in range(2)]
            self._peer_key = key
            self._peer_n = 0
        pb = self._peer[self._peer_n % 2]
        if not pb.ok:
            return None
        self._peer_n += 1
        rc = self.lib.hsseig_cauchy_sample_part_peers(gen.gen, self._leaf_of(part, w),
                                                      nat.ptr(om), ws, w, lo, hi,
                                                      nat.ptr(pb.ptrs[0]), nat.ptr(pb.ptrs[1]),
                                                      world, ws, nat.ptr(self.sample_work),
                                                      self._s())
        # past this point the other ranks store into our buffers: no NCCL fallback here
        nat.check(rc, "cauchy_sample_part_peers")
        peer_fence(group)
        return pb.local[0], pb.local[1]

    def build(self, gen, part, w, om, Y, Z, group=None, offdiag=True):
        """Construction; with several ranks each builds its subtrees below level log2(world),
        the subtree slots are all-gathered and the upper levels are built on every rank.
        offdiag: Y / Z are the off-diagonal sample (sample_part / sample_gather with part)."""
        from .hss import finish_construct
        from .secular import Status
        nat = self.nat
        tree = self.tree_for(part, w)
        tree.offdiag = bool(offdiag)
        tree._ranks = None
        st = Status(self.k)
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        args = (gen.gen, nat.ptr(om), om.shape[1], nat.ptr(Y), nat.ptr(Z), Y.shape[1], 1e-15,
                int(bool(offdiag)), ctypes.byref(tree.ct), nat.ptr(st.t))
        depth = tree.ct.depth
        if world > 1 and (1 << depth) >= world and (world & (world - 1)) == 0:
            s_lev = world.bit_length() - 1
            nat.check(self.lib.hsseig_tree_clear(ctypes.byref(tree.ct), self._s()), "tree_clear")
            nat.check(self.lib.hsseig_hss_build_rand_levels(*args, depth, s_lev, rank, world,
                                                            self._s()), "build_levels")
            gather_subtrees(tree, s_lev, group)
            nat.check(self.lib.hsseig_hss_build_rand_levels(*args, s_lev - 1, 0, 0, 1, self._s()),
                      "build_levels")
        else:
            nat.check(self.lib.hsseig_hss_build_rand(*args, self._s()), "hss_build_rand")
        tree._status = st
        finish_construct(tree)
        return tree

    def build_srrsc(self, gen, part, cap, tol, group=None):
        """ADC1 construction (csrc/srrsc.cu) partitioned like build(): each rank eliminates
        its subtrees below level log2(world), the node slots are all-gathered, the upper
        levels are built on every rank."""
        from .hss import HssTree, finish_construct
        from .secular import Status
        nat = self.nat
        tree = HssTree(part, cap)
        tree.method = "srrsc"
        need = int(self.lib.hsseig_srrsc_work_doubles(ctypes.byref(tree.ct)))
        if self._swork is None or self._swork.numel() < need:
            self._swork = torch.empty(need, dtype=torch.float64, device="cuda")
        st = Status(self.k)
        world = dist.get_world_size(group) if dist.is_initialized() else 1
        rank = dist.get_rank(group) if dist.is_initialized() else 0
        args = (gen.gen, float(tol), int(cap), ctypes.byref(tree.ct), nat.ptr(self._swork),
                nat.ptr(st.t))
        depth = tree.ct.depth
        if world > 1 and (1 << depth) >= world and (world & (world - 1)) == 0:
            s_lev = world.bit_length() - 1
            nat.check(self.lib.hsseig_tree_clear(ctypes.byref(tree.ct), self._s()), "tree_clear")
            nat.check(self.lib.hsseig_hss_build_srrsc_levels(*args, depth, s_lev, rank, world,
                                                             self._s()), "build_srrsc_levels")
            gather_subtrees(tree, s_lev, group)
            nat.check(self.lib.hsseig_hss_build_srrsc_levels(*args, s_lev - 1, 0, 0, 1,
                                                             self._s()), "build_srrsc_levels")
        else:
            nat.check(self.lib.hsseig_hss_build_srrsc(*args, self._s()), "hss_build_srrsc")
        tree._status = st
        finish_construct(tree)
        return tree

    def flagged(self, tree):
        return tree.flagged

    def construct_flops(self, tree):
        from .hss import _construct_flops, _srrsc_flops
        if getattr(tree, "method", "rand") == "srrsc":
            return _srrsc_flops(tree, tree.k)
        return _construct_flops(tree, tree.k, tree.w)

    def mult_flops(self, tree, P):
        from .hss import mult_flops
        return mult_flops(tree, P)

    def r_used(self, tree):
        return tree.r_used

    def multiply(self, X, tree):
        nat = self.nat
        if X.stride(0) % 2 or X.data_ptr() % 16:   # TMA rows: 16-byte aligned, even ld
            Xp = torch.empty(X.shape[0], X.shape[1] + (X.shape[1] & 1), dtype=torch.float64,
                             device="cuda")
            Xp[:, :X.shape[1]] = X
            X = Xp[:, :X.shape[1]]
        out = torch.empty(X.shape[0], self.k, dtype=torch.float64, device="cuda")
        need = int(self.lib.hsseig_matmul_work_doubles(X.shape[0], ctypes.byref(tree.ct)))
        if self._mwork is None or self._mwork.numel() < need:
            self._mwork = None
            self._mwork = torch.empty(need, dtype=torch.float64, device="cuda")
        nat.check(self.lib.hsseig_hss_matmul_right(nat.ptr(X), X.stride(0), X.shape[0],
                                                   ctypes.byref(tree.ct), nat.ptr(out), out.stride(0),
                                                   nat.ptr(self._mwork), self._s()), "hss_matmul_right")
        return out

    def dense(self, X, gen):
        return gen.right_multiply_into(X)

    # ---- distributed full solve (adc_solve_distributed)
    device = "cuda"

    def tensor(self, x):
        return torch.as_tensor(np.ascontiguousarray(x, dtype=np.float64), device="cuda")

    def local_solve(self, a, b, nodes, sub, cfg):
        from .solver import _plan, solve_subtree
        a_mod = nodes.split_diagonal(a, b)
        return solve_subtree(a_mod, b, nodes, sub, cfg)

    def deflate(self, nL, nR, L, zrow, bk):
        return deflate_merge(self.lib, nL, nR, L, zrow, bk)

    def assemble_rows(self, Qc, coff, nc, src, n):
        nat = self.nat
        W = torch.empty(Qc.shape[0], n, dtype=torch.float64, device="cuda")
        src_d = torch.as_tensor(src, device="cuda")
        nat.check(self.lib.hsseig_assemble_rows(nat.ptr(Qc), Qc.stride(0), Qc.shape[0], coff, nc,
                                                nat.ptr(src_d), n, nat.ptr(W), n, self._s()),
                  "assemble_rows")
        return W

    def rotate(self, W, ca, cb, c, s):
        nat = self.nat
        t = (torch.as_tensor(ca, device="cuda"), torch.as_tensor(cb, device="cuda"),
             self.tensor(c), self.tensor(s))
        nat.check(self.lib.hsseig_apply_rotations(nat.ptr(W), W.stride(0), W.shape[0],
                                                  *(nat.ptr(x) for x in t), len(ca), self._s()),
                  "apply_rotations")

    def gather(self, Qk, W, order, k):
        nat = self.nat
        n = W.shape[1]
        out = torch.empty_like(W)
        o = torch.as_tensor(np.ascontiguousarray(order, dtype=np.int64), device="cuda")
        A = Qk if Qk is not None else W
        nat.check(self.lib.hsseig_gather_columns(nat.ptr(A), A.stride(0), nat.ptr(W), W.stride(0), k,
                                                 nat.ptr(o), n, W.shape[0], nat.ptr(out), n,
                                                 self._s()), "gather")
        return out


def deflate_merge(lib, nL, nR, L, zrow, bk):
    """Host deflation of one merge (hsseig_wave_deflate with one merge): kept count,
    [kept | deflated] poles and weights, blockdiag column of every W column, rotations."""
    n = nL + nR
    P = lambda x: x.ctypes.data_as(ctypes.c_void_p)  # noqa: E731
    n1, n2 = np.array([nL], dtype=np.int64), np.array([nR], dtype=np.int64)
    roff = np.array([0, n], dtype=np.int64)
    L = np.ascontiguousarray(L, dtype=np.float64)
    zrow = np.ascontiguousarray(zrow, dtype=np.float64)
    bka = np.array([bk], dtype=np.float64)
    kept, rho = np.empty(1, dtype=np.int64), np.empty(1)
    d, z, src = np.empty(n), np.empty(n), np.empty(n, dtype=np.int64)
    rot_off = np.empty(2, dtype=np.int64)
    ca, cb, rc, rs = (np.empty(n, dtype=np.int64), np.empty(n, dtype=np.int64), np.empty(n),
                      np.empty(n))
    lib.hsseig_wave_deflate(1, P(n1), P(n2), P(roff), P(L), P(zrow), P(bka), P(kept), P(rho), P(d),
                            P(z), P(src), P(rot_off), P(ca), P(cb), P(rc), P(rs))
    nr = int(rot_off[1])
    return {"kept": int(kept[0]), "rho_eff": float(rho[0]), "d": d, "z": z, "src": src,
            "nrot": nr, "ca": ca[:nr], "cb": cb[:nr], "rc": rc[:nr], "rs": rs[:nr]}



# ----------------------------------------------------------------------------------------
# Multi-GPU full eigendecomposition (BASELINE config 5, SURVEY.md §8 e/f3)
# ----------------------------------------------------------------------------------------
_GROUPS = {}


def _group(ranks):
    """Process group of a contiguous rank range (created once, collectively)."""
    key = tuple(ranks)
    if key not in _GROUPS:
        _GROUPS[key] = dist.new_group(list(ranks))
    return _GROUPS[key]


def _split_a(a, b, nodes, max_depth):
    """Diagonal with the split modifications of the recursion nodes above max_depth."""
    return nodes.split_diagonal(a, b, max_depth)


def _gather_padded(vec, length, group, device):
    """All-gather 1-D tensors of up to `length` entries (padded); returns the list."""
    world = dist.get_world_size(group)
    t = torch.zeros(length, dtype=torch.float64, device=device)
    t[:vec.numel()] = vec
    parts = [torch.empty_like(t) for _ in range(world)]
    _all_gather(parts, t, group)
    return parts


class DistributedEigenResult:
    """Eigenvalues (replicated) and this rank's rows [row0, row1) of Q (all N columns)."""

    def __init__(self, lam, Q_rows, row0, row1, merges):
        self.lam, self.Q_rows, self.row0, self.row1, self.merges = lam, Q_rows, row0, row1, merges


def adc_solve_distributed(T, cfg, ops, group=None):
    """Full DC eigendecomposition over the ranks of `group` (a power of two, G = 2^g).

    Rank r solves the recursion subtree rooted at the r-th node of depth g alone (its
    base cases and merges, level-batched).  The merges above depth g are row-block
    sharded: every rank keeps its subtree's rows of the current eigenvector block for
    the whole ascent, so assembly, the Givens replay, the update (ShardedMerge: roots /
    weights / samples index-sharded and all-gathered, tree replicated or subtree-built,
    row-local multiply) and the final column gather are row-local.  Per merge only the
    two boundary rows (z) and the children's eigenvalues cross ranks.  The merge ids,
    seeds, deflation and records are the reference's (dc.py:174-257).
    """
    from .dc import MergeRecord
    from .solver import MAX_BASE, _tree
    # the same input checks as adc_solve (dc.py:185-186; solver.adc_solve)
    if not (np.all(np.isfinite(T.a)) and np.all(np.isfinite(T.b))):
        raise ValueError("matrix has non-finite entries")
    if cfg.base_size > MAX_BASE:
        raise ValueError(f"base_size above {MAX_BASE} is not supported by the device base case")
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    g = world.bit_length() - 1
    if world & (world - 1):
        raise ValueError("the distributed solver needs a power-of-two number of ranks")
    a = np.asarray(T.a, dtype=np.float64)
    b = np.asarray(T.b, dtype=np.float64)
    nodes, root = _tree(T.n, cfg.base_size)
    subs = sorted((i for i, nd in enumerate(nodes) if nd["depth"] == g), key=lambda i: nodes[i]["lo"])
    if len(subs) != world:
        raise ValueError("matrix too small for this many ranks (recursion shallower than log2 G)")
    granks = [dist.get_global_rank(group, r) for r in range(world)] if group is not None \
        else list(range(world))
    # groups of every merge above depth g (all ranks create all of them, in order)
    for d in range(g):
        size = 1 << (g - d)
        for j in range(1 << d):
            _group(granks[j * size:(j + 1) * size])
    me = subs[rank]
    lam, Qb, records = ops.local_solve(a, b, nodes, me, cfg)
    row0, row1 = nodes[me]["lo"], nodes[me]["hi"]
    cur = me
    parent = {}
    for i, nd in enumerate(nodes):
        if not nd["leaf"]:
            parent[nd["left"]] = i
            parent[nd["right"]] = i
    dev = ops.device
    for d in range(g - 1, -1, -1):
        P = parent[cur]
        nd = nodes[P]
        size = 1 << (g - d)
        j = rank // size
        ranks = granks[j * size:(j + 1) * size]
        grp = _group(ranks)
        half = size // 2
        left_side = (rank % size) < half
        nL, nR = nd["split"] - nd["lo"], nd["hi"] - nd["split"]
        n = nL + nR
        nmax = max(nL, nR)
        # children's eigenvalues and the boundary rows (last row of Q_L, first row of Q_R)
        lam_parts = _gather_padded(torch.as_tensor(lam, device=dev), nmax, grp, dev)
        lamL = lam_parts[0][:nL].cpu().numpy()
        lamR = lam_parts[half][:nR].cpu().numpy()
        edge = torch.zeros(2, nmax, dtype=torch.float64, device=dev)
        edge[0, :Qb.shape[1]] = Qb[0]
        edge[1, :Qb.shape[1]] = Qb[-1]
        eparts = [torch.empty_like(edge) for _ in range(size)]
        _all_gather(eparts, edge, grp)
        zrow = np.concatenate([eparts[half - 1][1, :nL].cpu().numpy(),
                               eparts[half][0, :nR].cpu().numpy()])
        bk = float(b[nd["split"] - 1])
        dfl = ops.deflate(nL, nR, np.concatenate([lamL, lamR]), zrow, bk)
        k, src = dfl["kept"], dfl["src"]
        rec = None
        if dfl["rho_eff"] != 0.0:
            rec = MergeRecord(size=n, kept=k, n_deflated=n - k)
            records[nd["mid"]] = rec
        W = ops.assemble_rows(Qb, 0 if left_side else nL, nL if left_side else nR, src, n)
        del Qb
        if dfl["nrot"]:
            ops.rotate(W, dfl["ca"], dfl["cb"], dfl["rc"], dfl["rs"])
        if k > 0:
            sm = ShardedMerge(k, cfg, ops, group=grp)
            lam_k, Qk, info = sm.run(ops.tensor(dfl["d"][:k]), ops.tensor(dfl["z"][:k]),
                                     dfl["rho_eff"], W[:, :k], seed=[cfg.seed, nd["mid"]],
                                     rows_total=n)
            lam_k = lam_k.cpu().numpy()
            if rec is not None:
                rec.used_hss = bool(info["used_hss"])
                rec.fell_back = bool(info["fell_back"])
                rec.hss_rank = int(info.get("r_used", 0))
                rec.flops = dict(info["flops"])
        else:
            lam_k, Qk = np.zeros(0), None
        lam_cat = np.concatenate([lam_k, dfl["d"][k:]])
        order = np.argsort(lam_cat, kind="stable")
        Qb = ops.gather(Qk, W, order, k)
        del W, Qk
        lam = lam_cat[order]
        cur = P
    # every rank reports the full merge list (its subtree's and the shared top merges)
    allrec = [None] * world
    dist.all_gather_object(allrec, records, group=group)
    merged = {}
    for r in allrec:
        merged.update(r)
    return DistributedEigenResult(lam, Qb, row0, row1, [merged[m] for m in sorted(merged)])
