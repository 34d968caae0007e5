"""Preallocated, low-synchronisation merge pipeline (the throughput path of dc.merge_update).

Same arithmetic and decisions as ``dc.merge_update`` + ``update_vectors_hss``
(pkg/src/hsseig/dc.py:141-171, 236-247), restructured for the device:

* buffers for roots, generators, samples, tree and multiply workspace are
  allocated once per (k, rows) and reused;
* the host synchronises only where the reference makes a data-dependent
  decision: after the secular solve (bracket check, partition and rank
  estimate, which need the pole gaps) and after the construction (the
  flag -> dense-fallback decision, where the Loewner radicand check is read too);
* the Gaussian sample is the reference's own draw default_rng([seed, merge_id])
  (hss.py:236), generated on the device bit-for-bit (sample_rng); if NumPy's
  ziggurat tables cannot be loaded the same draw is made on a host thread that
  starts with the merge.

Per-phase device times are taken with CUDA events on the launching stream.
"""
import concurrent.futures as cf
import ctypes
import os

import numpy as np
import torch

from . import _native as nat
from . import sample_rng
from .cauchy import CauchyEvecMatrix
from .flops import cauchy_eval_flops, gemm_flops, secular_flops
from .hss import (MAX_WIDTH, HssTree, _construct_flops, build_partition, finish_construct,
                  mult_flops, prefetch_construct, rank_bound)
from .secular import SecularConvergenceError, WeightRecomputationError

_POOL = cf.ThreadPoolExecutor(max_workers=1)
# SMs left to the upper levels' construction while the multiply's leaf up-level runs beside
# it (0: build, then multiply, in sequence)
SPLIT_RESERVE = int(os.environ.get("HSSEIG_SPLIT_RESERVE", "48"))
MAX_W = MAX_WIDTH
CHUNK = 1 << 18


def _ceil16(x):
    return (x + 15) // 16 * 16


class HostOmega:
    """Host fallback for the sample draw, produced on a thread into pinned memory.

    The row-major (k, w) block is the first k*w values of the generator's normal stream
    for every w, so generation starts before w is known and stops at the published k*w.
    """

    def __init__(self, n):
        self.buf = torch.empty(n, dtype=torch.float64, pin_memory=True)
        self.np = self.buf.numpy()
        self.target = n
        self.fut = None

    def start(self, seed):
        self.target = self.np.size
        self.fut = _POOL.submit(self._work, seed)

    def _work(self, seed):
        g = np.random.default_rng(seed)
        pos = 0
        while pos < self.target:
            n = min(CHUNK, self.target - pos)
            g.standard_normal(out=self.np[pos:pos + n])
            pos += n
        return pos

    def finish(self, count):
        self.target = count
        got = self.fut.result() if self.fut is not None else 0
        assert got >= count
        return self.buf[:count]


class MergePipeline:
    def __init__(self, k, cfg, rows, device_rng=True):
        nat.require_cuda()
        self.k, self.cfg, self.rows = int(k), cfg, int(rows)
        self.lib = nat.load()
        f64 = dict(dtype=torch.float64, device="cuda")
        k = self.k
        self.lam = torch.empty(k, **f64)
        self.gam = torch.empty(k, **f64)
        self.mu = torch.empty(k, **f64)
        self.dn = torch.empty(k, **f64)
        self.zh = torch.empty(k, **f64)
        self.v = torch.empty(k, **f64)
        self.its = torch.empty(k, dtype=torch.int32, device="cuda")
        self.swork = torch.empty(2 * k + 64, **f64)
        self.status = torch.zeros(8, dtype=torch.int64, device="cuda")
        self.h_status = torch.empty(8, dtype=torch.int64, pin_memory=True)
        self.h_mu = torch.empty(k, dtype=torch.float64, pin_memory=True)
        self.h_edges = torch.empty(3, dtype=torch.float64, pin_memory=True)
        wmax = _ceil16(MAX_W)
        self.Y = torch.empty(k * wmax, **f64)
        self.Z = torch.empty(k * wmax, **f64)
        self.om = torch.empty(k * wmax, **f64)
        self.om_flat = torch.empty(k * MAX_W, **f64)
        self.sample_work = torch.empty(int(self.lib.hsseig_sample_work_doubles(k, MAX_W)), **f64)
        self.device_rng = bool(device_rng) and sample_rng.available()
        if self.device_rng:
            self.normals = sample_rng.NormalStream(k * MAX_W)
        else:
            self.host_omega = HostOmega(k * MAX_W)
        self._tree_key = None
        self._mwork = None

    def _events(self, n):
        return [torch.cuda.Event(enable_timing=True) for _ in range(n)]

    def run(self, d, z, rho, X, seed, out=None, host_io=None, chunks=8):
        """One merge: returns a dict of phase times (ms), flops and decisions.

        host_io=(X_host, out_host): Q_old is streamed from pinned host memory into X in
        row chunks while the roots / sample / tree are computed, each chunk is multiplied
        as soon as it has landed and its rows of Q_new are copied back to out_host while
        the next chunk is multiplied (copy engines overlap the DMMA work).
        """
        lib, k, cfg = self.lib, self.k, self.cfg
        s = nat.stream_ptr()
        ev = self._events(7)
        ev[0].record()
        P = X.shape[0]
        if out is None:
            out = torch.empty(P, k, dtype=torch.float64, device="cuda")
        bounds = None
        if host_io is not None:
            Xh, Oh = host_io
            if not hasattr(self, "_h2d"):
                self._h2d, self._d2h = torch.cuda.Stream(), torch.cuda.Stream()
            bounds = [(P * i // chunks, P * (i + 1) // chunks) for i in range(chunks)]
            ev_in = []
            self._h2d.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self._h2d):
                for r0, r1 in bounds:
                    X[r0:r1].copy_(Xh[r0:r1], non_blocking=True)
                    e = torch.cuda.Event()
                    e.record(self._h2d)
                    ev_in.append(e)
        if self.device_rng:
            # the whole k x MAX_W prefix of the sample stream (the (k, w) block is its first
            # k*w values for every w), drawn before w is known on a side stream that
            # overlaps the root solve; tail records read back later
            if not hasattr(self, "_rng_stream"):
                self._rng_stream = torch.cuda.Stream()
            self._rng_stream.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(self._rng_stream):
                self.normals.draw(seed, k * MAX_W, self.om_flat)
                self._rng_done = torch.cuda.Event()
                self._rng_done.record(self._rng_stream)
        else:
            self.host_omega.start(seed)
        self.status.zero_()
        self.status[1:4] = k
        nat.check(lib.hsseig_secular(nat.ptr(d), nat.ptr(z), k, float(rho), nat.ptr(self.lam),
                                     nat.ptr(self.gam), nat.ptr(self.mu), nat.ptr(self.its),
                                     nat.ptr(self.swork), nat.ptr(self.status), s), "secular")
        nat.check(lib.hsseig_dnext(nat.ptr(d), nat.ptr(self.gam), nat.ptr(self.mu), k,
                                   nat.ptr(self.dn), s), "dnext")
        ev[1].record()
        # host needs: status (bracket), mu (partition shifts), span = lam[-1] - d[0]
        self.h_status.copy_(self.status, non_blocking=True)
        self.h_mu.copy_(self.mu, non_blocking=True)
        self.h_edges.copy_(torch.stack([d[0], d[-1], self.gam[-1]]), non_blocking=True)
        host_ready = torch.cuda.Event()
        host_ready.record()
        nat.check(lib.hsseig_loewner(nat.ptr(d), nat.ptr(self.dn), nat.ptr(self.gam),
                                     nat.ptr(self.mu), nat.ptr(z), k, float(rho), nat.ptr(self.zh),
                                     nat.ptr(self.status), s), "loewner")
        nat.check(lib.hsseig_normalizers(nat.ptr(d), nat.ptr(self.dn), nat.ptr(self.gam),
                                         nat.ptr(self.mu), nat.ptr(self.zh), k, nat.ptr(self.v), s),
                  "normalizers")
        ev[2].record()
        host_ready.synchronize()
        st = self.h_status.tolist()
        iters = int(st[0])
        bad = st[1] if st[1] < k else (st[2] if (k >= 2 and st[2] < k) else -1)
        if bad >= 0:
            raise SecularConvergenceError(f"root {bad} lost its bracket")
        info = {"flops": {}, "ms": {}, "used_hss": False, "fell_back": False, "r_used": 0,
                "device_rng": self.device_rng}
        fl_sec = secular_flops(k, iters) + 14 * k * k
        C = CauchyEvecMatrix(d, self.gam, self.mu, self.zh, self.v, dnext=self.dn)
        use_hss = cfg.method == "adc-rand" and k > cfg.hss_threshold
        tree = None
        fl_con = 0
        split = None
        if use_hss:
            mu_h = self.h_mu.numpy()
            try:
                part = build_partition(k, cfg.leaf_size, None, None, mu_h)
            except ValueError:
                part = None
            if part is not None:
                d0, dl, gl = self.h_edges.tolist()
                span = (dl + gl) - d0
                r_est = _rank_from(part, span, mu_h, cfg.rank_eps, cfg.rank_cap)
                r = min(r_est, part.min_leaf - cfg.oversample)
                w = r + cfg.oversample
                if r >= 1 and w <= MAX_W:
                    ws = _ceil16(w)
                    om = self.om[:k * ws].view(k, ws)
                    if self.device_rng:
                        try:
                            torch.cuda.current_stream().wait_event(self._rng_done)
                            self.normals.fixup()
                            om[:, :w].copy_(self.om_flat[:k * w].view(k, w))
                        except RuntimeError:   # unresolved rejection chain: the host draw
                            hv = np.random.default_rng(seed).standard_normal((k, w))
                            om[:, :w].copy_(torch.as_tensor(hv, device="cuda"))
                    else:
                        hv = self.host_omega.finish(k * w)
                        om[:, :w].copy_(hv.view(k, w), non_blocking=True)
                    tree = self._tree(part, w)
                    tree._status = _StatusView(self.status)
                    offdiag = getattr(cfg, "sample", "offdiag") == "offdiag"
                    tree.offdiag = offdiag
                    ev[3].record()
                    Y = self.Y[:k * ws].view(k, ws)
                    Z = self.Z[:k * ws].view(k, ws)
                    nat.check(lib.hsseig_cauchy_sample(C.gen, tree.ct.leaf_of if offdiag else None,
                                                       nat.ptr(om), ws, w, nat.ptr(Y), nat.ptr(Z), ws,
                                                       nat.ptr(self.sample_work), s), "cauchy_sample")
                    ev[4].record()
                    bargs = (C.gen, nat.ptr(om), ws, nat.ptr(Y), nat.ptr(Z), ws, float(1e-15),
                             int(offdiag), ctypes.byref(tree.ct), nat.ptr(self.status))
                    depth = tree.ct.depth
                    if bounds is None and SPLIT_RESERVE > 0 and depth >= 2:
                        # leaf level first; its up-sweep product G = X U_leaf then runs on a
                        # side stream (grid capped) beside the upper levels' construction
                        nat.check(lib.hsseig_tree_clear(ctypes.byref(tree.ct), s), "tree_clear")
                        nat.check(lib.hsseig_hss_build_rand_levels(*bargs, depth, depth, 0, 1, s),
                                  "hss_build_rand_levels")
                        split = self._leaf_up(X, out, tree)
                        nat.check(lib.hsseig_hss_build_rand_levels(*bargs, depth - 1, 0, 0, 1, s),
                                  "hss_build_rand_levels")
                    else:
                        nat.check(lib.hsseig_hss_build_rand(*bargs, s), "hss_build_rand")
                    ev[5].record()
        ev_m0 = torch.cuda.Event(enable_timing=True)
        pre = None
        if tree is not None and split is not None:
            # the leaf up-level already ran beside the construction: the rest of the product
            pre = prefetch_construct(tree, extra=[(self.status, self.h_status)])
            cur = torch.cuda.current_stream()
            cur.wait_event(split[2])
            ev_m0.record()
            nat.check(lib.hsseig_hss_matmul_right_part(nat.ptr(X), X.stride(0), X.shape[0],
                                                       ctypes.byref(tree.ct), nat.ptr(out),
                                                       out.stride(0), nat.ptr(self._mwork), 1, 0, s),
                      "hss_matmul_right_part")
            ev[6].record()
            finish_construct(tree, pre=pre)   # waits for the read-back: flags, ranks, r_used
            fl_con = _construct_flops(tree, k, w)
        elif tree is not None:
            # the multiply is queued right behind the construction and the async read-back of
            # its flags / ranks / the status block, before the host waits for that read-back
            # (the multiply's job table is built on the device from the ranks, its tiles
            # cover the sample width); a flagged tree (rare) is then replaced by the dense
            # fallback below, which overwrites out: the decision is the reference's
            # (dc.py:147-160), only its latency is hidden
            pre = prefetch_construct(tree, extra=[(self.status, self.h_status)])
            tree.ct.rmax = 0
            rows_max = P if bounds is None else max(r1 - r0 for r0, r1 in bounds)
            need = int(lib.hsseig_matmul_work_doubles(rows_max, ctypes.byref(tree.ct)))
            if self._mwork is None or self._mwork.numel() < need:
                self._mwork = None
                torch.cuda.empty_cache()
                self._mwork = torch.empty(need, dtype=torch.float64, device="cuda")
            ev_m0.record()
            if bounds is None:
                nat.check(lib.hsseig_hss_matmul_right(nat.ptr(X), X.stride(0), X.shape[0],
                                                      ctypes.byref(tree.ct), nat.ptr(out),
                                                      out.stride(0), nat.ptr(self._mwork), s),
                          "hss_matmul_right")
            else:
                cur = torch.cuda.current_stream()
                for (r0, r1), e in zip(bounds, ev_in):
                    cur.wait_event(e)
                    nat.check(lib.hsseig_hss_matmul_right(nat.ptr(X[r0:r1]), X.stride(0), r1 - r0,
                                                          ctypes.byref(tree.ct), nat.ptr(out[r0:r1]),
                                                          out.stride(0), nat.ptr(self._mwork), s),
                              "hss_matmul_right")
                    done = torch.cuda.Event()
                    done.record(cur)
                    self._d2h.wait_event(done)
                    with torch.cuda.stream(self._d2h):
                        Oh[r0:r1].copy_(out[r0:r1], non_blocking=True)
            ev[6].record()
            finish_construct(tree, pre=pre)   # waits for the read-back: flags, ranks, r_used
            fl_con = _construct_flops(tree, k, w)
        if not self.device_rng:
            self.host_omega.finish(0)
        st = self.h_status.tolist() if pre is not None else self.status.cpu().tolist()
        if st[3] < k:
            raise WeightRecomputationError(f"non-positive radicand at index {st[3]}")
        if tree is not None and not tree.flagged:
            info["used_hss"] = True
            info["r_used"] = tree.r_used
            fl_mult_local = mult_flops(tree, X.shape[0])
            fl_mult_full = mult_flops(tree, k)
            fl_dense = 0
        else:
            if bounds is not None:
                for e in ev_in:
                    torch.cuda.current_stream().wait_event(e)
            ev_m0 = torch.cuda.Event(enable_timing=True)
            ev_m0.record()
            C.right_multiply_into(X, out=out)
            ev[6].record()
            if bounds is not None:
                self._d2h.wait_stream(torch.cuda.current_stream())
                with torch.cuda.stream(self._d2h):
                    Oh.copy_(out, non_blocking=True)
            info["fell_back"] = use_hss
            fl_mult_local = fl_mult_full = 0
            fl_dense = cauchy_eval_flops(k * k) + gemm_flops(k, k, k)
        if bounds is not None:
            torch.cuda.current_stream().wait_stream(self._d2h)
        torch.cuda.synchronize()
        ms = {"secular": ev[0].elapsed_time(ev[1]),
              "loewner_normalizers": ev[1].elapsed_time(ev[2]),
              "multiply": ev_m0.elapsed_time(ev[6]),
              "total": ev[0].elapsed_time(ev[6])}
        if split is not None and info["used_hss"]:
            # kernel time of the product = its leaf up-level (side stream, beside the
            # construction) + the rest; the span is from the leaf up-level's start
            ms["multiply_leaf_up"] = split[1].elapsed_time(split[2])
            ms["multiply"] += ms["multiply_leaf_up"]
            ms["multiply_span"] = split[1].elapsed_time(ev[6])
        if info["used_hss"]:
            ms["host_partition_omega"] = ev[2].elapsed_time(ev[3])
            ms["sample"] = ev[3].elapsed_time(ev[4])
            ms["build"] = ev[4].elapsed_time(ev[5])
        info["ms"] = ms
        info["flops"] = {"secular": fl_sec, "hss_construct": fl_con,
                         "hss_mult_local": fl_mult_local, "hss_mult": fl_mult_full,
                         "update_dense": fl_dense}
        info["flops_total_fullP"] = fl_sec + fl_con + fl_mult_full + fl_dense
        info["iterations"] = iters
        return info

    def _leaf_up(self, X, out, tree):
        """Queue the multiply's leaf up-level on the side stream behind the leaf level of the
        construction (grid capped to leave SPLIT_RESERVE SMs to the upper levels); returns
        (stream, start event, done event)."""
        lib = self.lib
        P = X.shape[0]
        tree.ct.rmax = 0       # ranks not read back yet: tiles cover the sample width
        need = int(lib.hsseig_matmul_work_doubles(P, ctypes.byref(tree.ct)))
        if self._mwork is None or self._mwork.numel() < need:
            self._mwork = None
            torch.cuda.empty_cache()
            self._mwork = torch.empty(need, dtype=torch.float64, device="cuda")
        if not hasattr(self, "_mult_stream"):
            self._mult_stream = torch.cuda.Stream()
        side = self._mult_stream
        side.wait_stream(torch.cuda.current_stream())
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        sms = torch.cuda.get_device_properties(X.device).multi_processor_count
        with torch.cuda.stream(side):
            e0.record(side)
            nat.check(lib.hsseig_hss_matmul_right_part(nat.ptr(X), X.stride(0), P,
                                                       ctypes.byref(tree.ct), nat.ptr(out),
                                                       out.stride(0), nat.ptr(self._mwork), 0,
                                                       max(1, sms - SPLIT_RESERVE),
                                                       nat.stream_ptr(side)),
                      "hss_matmul_right_part")
            e1.record(side)
        return side, e0, e1

    def _tree(self, part, w):
        key = (part.ranges, w)
        if self._tree_key != key:
            self._treeobj = HssTree(part, w)
            self._tree_key = key
        t = self._treeobj
        t._ranks = None
        return t


class _StatusView:
    def __init__(self, t):
        self.t = t

    def read(self):
        return self.t.cpu().tolist()


def _rank_from(part, span, mu_h, eps, cap):
    """estimate_rank (hss.py:87-103) from host copies of the boundary gaps."""
    if part.n_leaves < 2:
        return 0
    r = 0
    for lo, _ in part.ranges[1:]:
        r = max(r, rank_bound(max(span / mu_h[lo - 1], 1.0), eps))
    return min(max(r, 1), cap)
