"""Device draw of the reference's Gaussian sample block (hss.py:236-237), bit-identical to NumPy.

``default_rng(seed).standard_normal((k, w))`` is NumPy's PCG64 stream through its
ziggurat.  The device kernels (csrc/normals.cu) need NumPy's ziggurat tables; they
are read from the installed NumPy extension module (the same build the reference
runs on), validated structurally, and the device output is compared with NumPy's
own draw once per process.  If any step fails, ``available()`` is False and
callers draw on the host with NumPy (the reference's own call).
"""
import ctypes
import glob
import os

import numpy as np
import torch

from . import _native as nat

_STATE = {"ok": None}
ZIG_R = 3.6541528853610088        # NumPy ziggurat_nor_r
ZIG_INV_R = 0.27366123732975828    # NumPy ziggurat_nor_inv_r
TAIL_CAP = 1 << 16
_KI0 = 0x000EF33D8025EF6A     # first entry of NumPy's ki_double table (ziggurat, 256 layers)


def _find_tables():
    import numpy.random as npr
    for path in glob.glob(os.path.join(os.path.dirname(npr.__file__), "_generator*.so")):
        blob = open(path, "rb").read()
        for off in range(8):
            uu = np.frombuffer(blob[off: off + (len(blob) - off) // 8 * 8], dtype="<u8")
            for i in np.flatnonzero(uu == _KI0):
                start = off + 8 * int(i)
                if start < 4096 or start + 2048 > len(blob):
                    continue
                ki = np.frombuffer(blob[start: start + 2048], dtype="<u8").copy()
                wi = np.frombuffer(blob[start - 2048: start], dtype="<f8").copy()
                fi = np.frombuffer(blob[start - 4096: start - 2048], dtype="<f8").copy()
                if (ki[1] == 0 and fi[0] == 1.0 and np.all(np.diff(fi) < 0)
                        and 8.6e-16 < wi[0] < 8.7e-16 and np.all(wi[1:] > 0)):
                    return ki, wi, fi
    return None


def pcg_state(seed):
    """(state_hi, state_lo, inc_hi, inc_lo) of default_rng(seed)'s PCG64."""
    st = np.random.default_rng(seed).bit_generator.state["state"]
    s, inc = int(st["state"]), int(st["inc"])
    m = (1 << 64) - 1
    return s >> 64, s & m, inc >> 64, inc & m


def available():
    if _STATE["ok"] is None:
        _STATE["ok"] = False
        try:
            tabs = _find_tables()
            if tabs is not None and torch.cuda.is_available():
                lib = nat.load()
                ki, wi, fi = tabs
                nat.check(lib.hsseig_set_normal_tables(ki.ctypes.data_as(ctypes.c_void_p),
                                                       wi.ctypes.data_as(ctypes.c_void_p),
                                                       fi.ctypes.data_as(ctypes.c_void_p)),
                          "set_normal_tables")
                _STATE["ok"] = True
                n = 300_000
                got = normals([7, 11], n).cpu().numpy()
                _STATE["ok"] = bool(np.array_equal(
                    got, np.random.default_rng([7, 11]).standard_normal(n)))
        except (OSError, RuntimeError, ValueError):
            _STATE["ok"] = False
    return _STATE["ok"]


class NormalStream:
    """Reusable device buffers for sample draws up to nmax values."""

    def __init__(self, nmax):
        self.lib = nat.load()
        self.nmax = int(nmax)
        self.work = torch.empty(int(self.lib.hsseig_normals_work_bytes(self.nmax)),
                                dtype=torch.uint8, device="cuda")
        self.fail = torch.zeros(1, dtype=torch.int32, device="cuda")
        self.tails = torch.zeros(1 + 3 * TAIL_CAP, dtype=torch.int64, device="cuda")
        self.h_tails = torch.empty(1 + 3 * TAIL_CAP, dtype=torch.int64, pin_memory=True)
        self.h_fail = torch.empty(1, dtype=torch.int32, pin_memory=True)
        self.h_pairs = torch.empty(2 * TAIL_CAP, dtype=torch.int64, pin_memory=True)
        self.d_pairs = torch.empty(2 * TAIL_CAP, dtype=torch.int64, device="cuda")
        self._ev = None
        self._fix_ev = None

    def draw(self, seed, n, out, w=None, ld=None, state=None):
        """Enqueue the first n normals of default_rng(seed) into out (device float64).

        With w / ld the values land as the row-major (n / w) x w block with leading
        dimension ld, i.e. standard_normal((n // w, w)) in a padded layout.
        """
        if n > self.nmax:
            raise ValueError("draw longer than the stream buffers")
        w = int(w or max(n, 1))
        ld = int(ld or w)
        sh, sl, ih, il = state if state is not None else pcg_state(seed)
        self.fail.zero_()
        nat.check(self.lib.hsseig_pcg64_normals(sh, sl, ih, il, int(n), w, ld, nat.ptr(out),
                                                nat.ptr(self.work), nat.ptr(self.fail),
                                                nat.ptr(self.tails), TAIL_CAP, nat.stream_ptr()),
                  "pcg64_normals")
        # the tail records and the failure flag come back asynchronously; fixup() applies them
        self.h_tails.copy_(self.tails, non_blocking=True)
        self.h_fail.copy_(self.fail, non_blocking=True)
        self._ev = torch.cuda.Event()
        self._ev.record()
        self._out = out
        return out

    def fixup(self):
        """Re-evaluate the ziggurat-tail values with the C library's log1p (as NumPy does).

        Waits for the draw's record read-back (not for the whole stream)."""
        self._ev.synchronize()
        if int(self.h_fail[0]):
            raise RuntimeError("device normal stream could not resolve the rejection chain")
        if self._fix_ev is not None:      # the previous fix-up's upload has left h_pairs
            self._fix_ev.synchronize()
        # host C (the C library's log1p, as NumPy) + one ordered upload + scatter kernel
        cnt = int(self.lib.hsseig_normals_fixup(nat.ptr(self.h_tails), TAIL_CAP, ZIG_R, ZIG_INV_R,
                                                nat.ptr(self.h_pairs), nat.ptr(self.d_pairs),
                                                nat.ptr(self._out), nat.stream_ptr()))
        if cnt < 0:
            nat.check(-cnt, "normals_fixup")
        self._fix_ev = torch.cuda.Event()
        self._fix_ev.record()
        return cnt

    def failed(self):
        self._ev.synchronize()
        return bool(int(self.h_fail[0]))


def normals(seed, n):
    """First n values of default_rng(seed).standard_normal, drawn on the device."""
    out = torch.empty(int(n), dtype=torch.float64, device="cuda")
    ns = NormalStream(n)
    ns.draw(seed, n, out)
    ns.fixup()
    return out
