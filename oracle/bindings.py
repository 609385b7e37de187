"""ctypes bindings for the two CPU checkers (TEST INFRASTRUCTURE ONLY).

Both libraries take plain fp64 / int64 row-major buffers; these wrappers take
and return numpy arrays.  ``orc`` is the C restatement, ``ref`` the reference
compiled from its own sources.  Everything is fp64 like the reference
(matrix.hpp:12-14).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORC_SO = os.path.join(HERE, "_build", "liborc.so")
REF_SO = os.path.join(HERE, "_ref", "libfmoe_ref.so")
REF_SRC = "/root/reference/proj"

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int64, flags="C_CONTIGUOUS")
_i64 = C.c_int64
_u64 = C.c_uint64
_vp = C.c_void_p


def build(force: bool = False) -> None:
    """Compile the oracle (always) and oracle/_ref (only when the reference
    sources are present, i.e. in the build container)."""
    targets = ["orc"]
    if os.path.isdir(os.path.join(REF_SRC, "src")):
        targets.append("ref")
    cmd = ["make", "-s", "-C", HERE] + (["-B"] if force else []) + targets
    subprocess.run(cmd, check=True)


class CheckerError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _arr(a, dtype):
    return np.ascontiguousarray(a, dtype=dtype)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_vp)


class _Lib:
    def __init__(self, path: str, err_fn: str):
        self.path = path
        self._lib = None
        self._err = err_fn

    @property
    def lib(self):
        if self._lib is None:
            if not os.path.exists(self.path):
                if self.path == ORC_SO:
                    build()
                else:
                    raise FileNotFoundError(self.path)
            self._lib = C.CDLL(self.path)
            getattr(self._lib, self._err).restype = C.c_char_p
        return self._lib

    def check(self, rc: int):
        if rc != 0:
            raise CheckerError(rc, getattr(self.lib, self._err)().decode())

    def call(self, name, *args, restype=C.c_int):
        fn = getattr(self.lib, name)
        fn.restype = restype
        conv = []
        for a in args:
            if isinstance(a, np.ndarray):
                conv.append(a.ctypes.data_as(_vp))
            elif a is None:
                conv.append(None)
            elif isinstance(a, float):
                conv.append(C.c_double(a))
            else:
                conv.append(_i64(int(a)))
        rc = fn(*conv)
        if restype is C.c_int:
            self.check(rc)
        return rc


class Orc(_Lib):
    """fmoe_oracle.c"""

    def __init__(self):
        super().__init__(ORC_SO, "orc_last_error")

    def stream_seed(self, base: int, stream: int) -> int:
        f = self.lib.orc_stream_seed
        f.restype, f.argtypes = _u64, [_u64, _u64]
        return int(f(base, stream))

    def uniform_fill(self, seed: int, n: int, lo=-1.0, hi=1.0) -> np.ndarray:
        out = np.empty(n, np.float64)
        f = self.lib.orc_uniform_fill
        f.restype, f.argtypes = None, [_u64, _vp, _i64, C.c_double, C.c_double]
        f(seed, _ptr(out), n, lo, hi)
        return out

    def seeded_matrix(self, seed, stream, rows, cols, lo=-1.0, hi=1.0):
        """fmoe_bench.cpp:128-134 seeded_matrix."""
        return self.uniform_fill(self.stream_seed(seed, stream), rows * cols, lo, hi).reshape(rows, cols)

    def init_state(self, seed, d, h, e, e_first=0, e_count=None):
        """init_state (moe_layer.cpp:28-45) -> dict of fp64 weights for experts
        [e_first, e_first+e_count) (global indices) and the gate over e experts."""
        e_count = e if e_count is None else e_count
        wg = np.empty((d, e), np.float64)
        f = self.lib.orc_init_gate
        f.restype, f.argtypes = None, [_u64, _i64, _i64, _vp]
        f(seed, d, e, _ptr(wg))
        w1 = np.empty((e_count, d, h)); b1 = np.empty((e_count, h))
        w2 = np.empty((e_count, h, d)); b2 = np.empty((e_count, d))
        g = self.lib.orc_init_expert
        g.restype, g.argtypes = None, [_u64, _u64, _i64, _i64, _vp, _vp, _vp, _vp]
        for i in range(e_count):
            g(seed, e_first + i, d, h, _ptr(w1[i]), _ptr(b1[i]), _ptr(w2[i]), _ptr(b2[i]))
        return dict(wg=wg, w1=w1, b1=b1, w2=w2, b2=b2)

    def matmul(self, a, b):
        a, b = _arr(a, np.float64), _arr(b, np.float64)
        out = np.empty((a.shape[0], b.shape[1]))
        f = self.lib.orc_matmul
        f.restype = None
        f(_ptr(a), _ptr(b), _ptr(out), _i64(a.shape[0]), _i64(a.shape[1]), _i64(b.shape[1]))
        return out

    def softmax_rows(self, a):
        a = _arr(a, np.float64)
        out = np.empty_like(a)
        f = self.lib.orc_softmax_rows
        f.restype = None
        f(_ptr(a), _ptr(out), _i64(a.shape[0]), _i64(a.shape[1]))
        return out

    def topk_rows(self, a, k):
        a = _arr(a, np.float64)
        idx = np.empty((a.shape[0], k), np.int64)
        vals = np.empty((a.shape[0], k))
        self.call("orc_topk_rows", a, a.shape[0], a.shape[1], k, idx, vals)
        return idx, vals

    def gate_forward(self, x, wg, k, want_logits=False):
        x, wg = _arr(x, np.float64), _arr(wg, np.float64)
        n, d = x.shape
        e = wg.shape[1]
        logits = np.empty((n, e))
        scores = np.empty((n, e))
        idx = np.empty((n, k), np.int64)
        vals = np.empty((n, k))
        self.call("orc_gate_forward", x, wg, n, d, e, k, logits, scores, idx, vals)
        if want_logits:
            return scores, idx, vals, logits
        return scores, idx, vals

    def gate_dlogits(self, scores, idx, d_topk):
        scores, idx, d_topk = _arr(scores, np.float64), _arr(idx, np.int64), _arr(d_topk, np.float64)
        n, e = scores.shape
        out = np.empty((n, e))
        f = self.lib.orc_gate_dlogits
        f.restype = None
        f(_ptr(scores), _ptr(idx), _ptr(d_topk), _i64(n), _i64(e), _i64(idx.shape[1]), _ptr(out))
        return out

    def gate_backward(self, x, wg, scores, idx, d_topk):
        x, wg = _arr(x, np.float64), _arr(wg, np.float64)
        scores, idx, d_topk = _arr(scores, np.float64), _arr(idx, np.int64), _arr(d_topk, np.float64)
        n, d = x.shape
        e = wg.shape[1]
        d_wg = np.empty((d, e))
        d_x = np.empty((n, d))
        f = self.lib.orc_gate_backward
        f.restype = None
        f(_ptr(x), _ptr(wg), _ptr(scores), _ptr(idx), _ptr(d_topk), _i64(n), _i64(d), _i64(e),
          _i64(idx.shape[1]), _ptr(d_wg), _ptr(d_x))
        return d_wg, d_x

    def build_plan(self, idx, num_experts):
        idx = _arr(idx, np.int64)
        n, k = idx.shape
        counts = np.empty(num_experts, np.int64)
        offsets = np.empty(num_experts, np.int64)
        src = np.empty(n * k, np.int64)
        slot = np.empty(n * k, np.int64)
        inv = np.empty((n, k), np.int64)
        self.call("orc_build_plan", idx, n, k, num_experts, counts, offsets, src, slot, inv)
        return dict(counts=counts, offsets=offsets, src_row=src, slot=slot, inverse_pos=inv)

    def scatter(self, x, plan):
        x = _arr(x, np.float64)
        src = plan["src_row"]
        out = np.empty((src.shape[0], x.shape[1]))
        f = self.lib.orc_scatter
        f.restype = None
        f(_ptr(x), _ptr(src), _i64(src.shape[0]), _i64(x.shape[1]), _ptr(out))
        return out

    def gather_combine(self, ys, plan, w):
        ys, w = _arr(ys, np.float64), _arr(w, np.float64)
        inv = plan["inverse_pos"]
        n, k = inv.shape
        out = np.empty((n, ys.shape[1]))
        f = self.lib.orc_gather_combine
        f.restype = None
        f(_ptr(ys), _ptr(inv), _ptr(w), _i64(n), _i64(k), _i64(ys.shape[1]), _ptr(out))
        return out

    def scatter_backward(self, d_xs, plan):
        d_xs = _arr(d_xs, np.float64)
        inv = plan["inverse_pos"]
        n, k = inv.shape
        out = np.empty((n, d_xs.shape[1]))
        f = self.lib.orc_scatter_backward
        f.restype = None
        f(_ptr(d_xs), _ptr(inv), _i64(n), _i64(k), _i64(d_xs.shape[1]), _ptr(out))
        return out

    def gather_combine_backward(self, d_y, ys, plan, w):
        d_y, ys, w = _arr(d_y, np.float64), _arr(ys, np.float64), _arr(w, np.float64)
        inv = plan["inverse_pos"]
        n, k = inv.shape
        d = ys.shape[1]
        d_ys = np.empty_like(ys)
        d_w = np.empty((n, k))
        f = self.lib.orc_gather_combine_backward
        f.restype = None
        f(_ptr(d_y), _ptr(ys), _ptr(inv), _ptr(w), _i64(n), _i64(k), _i64(d), _ptr(d_ys), _ptr(d_w))
        return d_ys, d_w

    def expert_forward(self, x, w1, b1, w2, b2):
        x = _arr(x, np.float64)
        rows, d = x.shape
        h = w1.shape[1]
        y = np.empty((rows, d)); pre = np.empty((rows, h)); hid = np.empty((rows, h))
        f = self.lib.orc_expert_forward
        f.restype = None
        f(_ptr(x), _i64(rows), _ptr(_arr(w1, np.float64)), _ptr(_arr(b1, np.float64)),
          _ptr(_arr(w2, np.float64)), _ptr(_arr(b2, np.float64)), _i64(d), _i64(h),
          _ptr(y), _ptr(pre), _ptr(hid))
        return y, pre, hid

    def expert_backward(self, d_y, x, pre, hid, w1, w2):
        rows, d = x.shape
        h = w1.shape[1]
        d_x = np.empty((rows, d)); dw1 = np.empty((d, h)); db1 = np.empty(h)
        dw2 = np.empty((h, d)); db2 = np.empty(d)
        f = self.lib.orc_expert_backward
        f.restype = None
        args = [_arr(d_y, np.float64), _arr(x, np.float64), _arr(pre, np.float64), _arr(hid, np.float64)]
        f(*[_ptr(a) for a in args], _i64(rows), _ptr(_arr(w1, np.float64)), _ptr(_arr(w2, np.float64)),
          _i64(d), _i64(h), _ptr(d_x), _ptr(dw1), _ptr(db1), _ptr(dw2), _ptr(db2))
        return d_x, dict(dw1=dw1, db1=db1, dw2=dw2, db2=db2)

    def moe_forward_backward(self, x, dy, k, wg, w1, b1, w2, b2):
        x = _arr(x, np.float64)
        n, d = x.shape
        e, _, h = w1.shape
        y = np.empty((n, d)); idx = np.empty((n, k), np.int64); scores = np.empty((n, e))
        out = dict(y=y, idx=idx, scores=scores)
        if dy is not None:
            dy = _arr(dy, np.float64)
            out.update(dx=np.empty((n, d)), dwg=np.empty((d, e)), dw1=np.empty((e, d, h)),
                       db1=np.empty((e, h)), dw2=np.empty((e, h, d)), db2=np.empty((e, d)))
        g = lambda key: out.get(key)  # noqa: E731
        self.call("orc_moe_forward_backward", x, dy, n, d, h, e, k, _arr(wg, np.float64),
                  _arr(w1, np.float64), _arr(b1, np.float64), _arr(w2, np.float64),
                  _arr(b2, np.float64), y, idx, scores, g("dx"), g("dwg"), g("dw1"), g("db1"),
                  g("dw2"), g("db2"))
        return out

    def exchange_counts(self, local_counts):
        lc = _arr(local_counts, np.int64)
        world, total = lc.shape
        out = np.empty((world, world, total // world), np.int64)
        self.call("orc_exchange_counts", lc, world, total, out)
        return out

    def all_to_all_rows(self, send_bufs, local_counts, rank):
        """collectives.cpp:146-203 for `rank`, given every rank's send buffer."""
        lc = _arr(local_counts, np.int64)
        world, total = lc.shape
        bufs = [_arr(b, np.float64) for b in send_bufs]
        d = bufs[0].shape[1]
        el = total // world
        rows = int(sum(lc[s, rank * el:(rank + 1) * el].sum() for s in range(world)))
        out = np.empty((rows, d))
        ptrs = (C.c_void_p * world)(*[b.ctypes.data for b in bufs])
        f = self.lib.orc_all_to_all_rows
        f.restype = None
        f(ptrs, _ptr(lc), _i64(world), _i64(total), _i64(rank), _i64(d), _ptr(out))
        return out


class Ref(_Lib):
    """The reference compiled from /root/reference/proj/src (namespace fmoe_ref)."""

    def __init__(self):
        super().__init__(REF_SO, "ref_last_error")

    def stream_seed(self, base, stream):
        f = self.lib.ref_stream_seed
        f.restype, f.argtypes = _u64, [_u64, _u64]
        return int(f(base, stream))

    def uniform_fill(self, seed, n, lo=-1.0, hi=1.0):
        out = np.empty(n)
        f = self.lib.ref_uniform_fill
        f.restype, f.argtypes = None, [_u64, _vp, _i64, C.c_double, C.c_double]
        f(seed, _ptr(out), n, lo, hi)
        return out

    def save_checkpoint(self, path, w, n_b=0, k=1, n_e_local=None, world=1, seed=0):
        """save_checkpoint (checkpoint.cpp:63-92) of the weight dict w."""
        e, d, h = w["w1"].shape
        meta = np.array([n_b, k, e if n_e_local is None else n_e_local, world, seed], np.int64)
        f = self.lib.ref_save_checkpoint
        f.restype = C.c_int
        f.argtypes = [C.c_char_p, _i64, _i64, _i64] + [_vp] * 6
        self.check(f(path.encode(), d, h, e, _ptr(meta),
                     *[_ptr(_arr(w[key], np.float64)) for key in ("wg", "w1", "b1", "w2", "b2")]))

    def load_checkpoint(self, path):
        """load_checkpoint (checkpoint.cpp:94-122) -> (header dict, weight dict)."""
        f = self.lib.ref_load_checkpoint
        f.restype = C.c_int
        f.argtypes = [C.c_char_p] + [_vp] * 6
        hd = np.zeros(7, np.int64)
        self.check(f(path.encode(), _ptr(hd), None, None, None, None, None))
        n_b, d, h, k, el, world, seed = (int(v) for v in hd)
        e = el * world
        w = dict(wg=np.empty((d, e)), w1=np.empty((e, d, h)), b1=np.empty((e, h)), w2=np.empty((e, h, d)),
                 b2=np.empty((e, d)))
        self.check(f(path.encode(), _ptr(hd), *[_ptr(w[key]) for key in ("wg", "w1", "b1", "w2", "b2")]))
        return dict(n_b=n_b, d_m=d, d_h=h, k=k, n_e_local=el, world_size=world, seed=seed), w

    def init_state(self, seed, d, h, e, k=1):
        wg = np.empty((d, e)); w1 = np.empty((e, d, h)); b1 = np.empty((e, h))
        w2 = np.empty((e, h, d)); b2 = np.empty((e, d))
        f = self.lib.ref_init_state
        f.restype = C.c_int
        f.argtypes = [_u64, _i64, _i64, _i64, _i64] + [_vp] * 5
        self.check(f(seed, d, h, e, k, *[_ptr(a) for a in (wg, w1, b1, w2, b2)]))
        return dict(wg=wg, w1=w1, b1=b1, w2=w2, b2=b2)

    def matmul(self, a, b):
        a, b = _arr(a, np.float64), _arr(b, np.float64)
        out = np.empty((a.shape[0], b.shape[1]))
        self.call("ref_matmul", a, b, out, a.shape[0], a.shape[1], b.shape[1])
        return out

    def softmax_rows(self, a):
        a = _arr(a, np.float64)
        out = np.empty_like(a)
        self.call("ref_softmax_rows", a, out, a.shape[0], a.shape[1])
        return out

    def topk_rows(self, a, k):
        a = _arr(a, np.float64)
        idx = np.empty((a.shape[0], k), np.int64)
        vals = np.empty((a.shape[0], k))
        self.call("ref_topk_rows", a, a.shape[0], a.shape[1], k, idx, vals)
        return idx, vals

    def gate_forward(self, x, wg, k):
        x, wg = _arr(x, np.float64), _arr(wg, np.float64)
        n, d = x.shape
        e = wg.shape[1]
        scores = np.empty((n, e)); idx = np.empty((n, k), np.int64); vals = np.empty((n, k))
        self.call("ref_gate_forward", x, wg, n, d, e, k, scores, idx, vals)
        return scores, idx, vals

    def gate_backward(self, x, wg, scores, idx, vals, d_topk):
        x, wg = _arr(x, np.float64), _arr(wg, np.float64)
        n, d = x.shape
        e = wg.shape[1]
        k = idx.shape[1]
        d_wg = np.empty((d, e)); d_x = np.empty((n, d))
        self.call("ref_gate_backward", x, wg, _arr(scores, np.float64), _arr(idx, np.int64),
                  _arr(vals, np.float64), _arr(d_topk, np.float64), n, d, e, k, d_wg, d_x)
        return d_wg, d_x

    def build_plan(self, idx, num_experts):
        idx = _arr(idx, np.int64)
        n, k = idx.shape
        counts = np.empty(num_experts, np.int64); offsets = np.empty(num_experts, np.int64)
        src = np.empty(n * k, np.int64); slot = np.empty(n * k, np.int64)
        inv = np.empty((n, k), np.int64)
        self.call("ref_build_plan", idx, n, k, num_experts, counts, offsets, src, slot, inv)
        return dict(counts=counts, offsets=offsets, src_row=src, slot=slot, inverse_pos=inv)

    def scatter(self, x, idx, num_experts):
        x, idx = _arr(x, np.float64), _arr(idx, np.int64)
        n, k = idx.shape
        out = np.empty((n * k, x.shape[1]))
        self.call("ref_scatter", x, idx, n, k, num_experts, x.shape[1], out)
        return out

    def gather_combine(self, ys, idx, w, num_experts):
        ys, idx, w = _arr(ys, np.float64), _arr(idx, np.int64), _arr(w, np.float64)
        n, k = idx.shape
        out = np.empty((n, ys.shape[1]))
        self.call("ref_gather_combine", ys, idx, w, n, k, num_experts, ys.shape[1], out)
        return out

    def scatter_backward(self, d_xs, idx, num_experts):
        d_xs, idx = _arr(d_xs, np.float64), _arr(idx, np.int64)
        n, k = idx.shape
        out = np.empty((n, d_xs.shape[1]))
        self.call("ref_scatter_backward", d_xs, idx, n, k, num_experts, d_xs.shape[1], out)
        return out

    def gather_combine_backward(self, d_y, ys, idx, w, num_experts):
        d_y, ys, idx, w = (_arr(d_y, np.float64), _arr(ys, np.float64), _arr(idx, np.int64),
                           _arr(w, np.float64))
        n, k = idx.shape
        d_ys = np.empty_like(ys); d_w = np.empty((n, k))
        self.call("ref_gather_combine_backward", d_y, ys, idx, w, n, k, num_experts, ys.shape[1],
                  d_ys, d_w)
        return d_ys, d_w

    def multi_expert(self, xs, counts, w1, b1, w2, b2, d_ys=None):
        xs = _arr(xs, np.float64)
        counts = _arr(counts, np.int64)
        e, d, h = w1.shape
        rows = xs.shape[0]
        ys = np.empty((rows, d))
        out = dict(ys=ys)
        if d_ys is not None:
            out.update(d_xs=np.empty((rows, d)), dw1=np.empty((e, d, h)), db1=np.empty((e, h)),
                       dw2=np.empty((e, h, d)), db2=np.empty((e, d)))
            d_ys = _arr(d_ys, np.float64)
        g = out.get
        self.call("ref_multi_expert", xs, counts, e, d, h, _arr(w1, np.float64), _arr(b1, np.float64),
                  _arr(w2, np.float64), _arr(b2, np.float64), d_ys, ys, g("d_xs"), g("dw1"),
                  g("db1"), g("dw2"), g("db2"))
        return out

    def moe_forward_backward(self, x, dy, k, wg, w1, b1, w2, b2):
        x = _arr(x, np.float64)
        n, d = x.shape
        e, _, h = w1.shape
        out = dict(y=np.empty((n, d)), idx=np.empty((n, k), np.int64))
        if dy is not None:
            dy = _arr(dy, np.float64)
            out.update(dx=np.empty((n, d)), dwg=np.empty((d, e)), dw1=np.empty((e, d, h)),
                       db1=np.empty((e, h)), dw2=np.empty((e, h, d)), db2=np.empty((e, d)))
        g = out.get
        self.call("ref_moe_forward_backward", x, dy, n, d, h, e, k, _arr(wg, np.float64),
                  _arr(w1, np.float64), _arr(b1, np.float64), _arr(w2, np.float64),
                  _arr(b2, np.float64), out["y"], out["idx"], g("dx"), g("dwg"), g("dw1"),
                  g("db1"), g("dw2"), g("db2"))
        return out

    def naive_forward(self, x, k, wg, w1, b1, w2, b2):
        x = _arr(x, np.float64)
        n, d = x.shape
        e, _, h = w1.shape
        y = np.empty((n, d))
        self.call("ref_naive_forward", x, n, d, h, e, k, _arr(wg, np.float64), _arr(w1, np.float64),
                  _arr(b1, np.float64), _arr(w2, np.float64), _arr(b2, np.float64), y)
        return y

    def moe_distributed(self, x, dy, world, k, wg, w1, b1, w2, b2):
        """x/dy are the rank-major concatenation [world*n, d]."""
        x = _arr(x, np.float64)
        nt, d = x.shape
        n = nt // world
        e, _, h = w1.shape
        el = e // world
        out = dict(y=np.empty((nt, d)), send_counts=np.empty((world, e), np.int64),
                   recv_counts=np.empty((world, e), np.int64))
        if dy is not None:
            dy = _arr(dy, np.float64)
            out.update(dx=np.empty((nt, d)), dwg=np.empty((world, d, e)), dw1=np.empty((e, d, h)),
                       db1=np.empty((e, h)), dw2=np.empty((e, h, d)), db2=np.empty((e, d)))
        g = out.get
        self.call("ref_moe_distributed", x, dy, world, n, d, h, el, k, _arr(wg, np.float64),
                  _arr(w1, np.float64), _arr(b1, np.float64), _arr(w2, np.float64),
                  _arr(b2, np.float64), out["y"], g("dx"), g("dwg"), g("dw1"), g("db1"), g("dw2"),
                  g("db2"), out["send_counts"], out["recv_counts"])
        return out

    def toy_task(self, n, d, h, k, e_local, world, seed):
        """make_toy_task -> (inputs, targets), [n*world, d] each."""
        x = np.empty((n * world, d))
        t = np.empty((n * world, d))
        f = self.lib.ref_toy_task
        f.restype = C.c_int
        f.argtypes = [_i64] * 6 + [_u64, _vp, _vp]
        self.check(f(n, d, h, k, e_local, world, seed, _ptr(x), _ptr(t)))
        return x, t

    def train_steps(self, x, target, world, n, h, e_local, k, seed, steps, lr):
        """ref_train_steps: the reference's train_step trajectory (x/target are
        the rank-major [world*n, d] task)."""
        x, target = _arr(x, np.float64), _arr(target, np.float64)
        d = x.shape[1]
        e = e_local * world
        out = dict(losses=np.empty(steps), wg=np.empty((d, e)), w1=np.empty((e, d, h)), b1=np.empty((e, h)),
                   w2=np.empty((e, h, d)), b2=np.empty((e, d)))
        f = self.lib.ref_train_steps
        f.restype = C.c_int
        f.argtypes = [_i64] * 6 + [_u64, _i64, C.c_double] + [_vp] * 8
        self.check(f(world, n, d, h, e_local, k, seed, steps, lr, _ptr(x), _ptr(target),
                     *[_ptr(out[key]) for key in ("losses", "wg", "w1", "b1", "w2", "b2")]))
        return out

    def exchange_counts(self, local_counts):
        lc = _arr(local_counts, np.int64)
        world, total = lc.shape
        out = np.empty((world, total), np.int64)
        self.call("ref_exchange_counts", lc, world, total, out)
        return out.reshape(world, world, total // world)


orc = Orc()
ref = Ref()


def ref_available() -> bool:
    return os.path.exists(REF_SO)


REF_SO_V4 = os.path.join(HERE, "_ref", "libfmoe_ref_v4.so")


def host_has_avx512() -> bool:
    try:
        flags = open("/proc/cpuinfo").read().split("flags", 2)[1].split("\n", 1)[0].split()
    except (OSError, IndexError):
        return False
    return all(f in flags for f in ("avx512f", "avx512bw", "avx512cd", "avx512dq", "avx512vl"))


def ref_timing_so() -> tuple[str, str]:
    """The reference build to TIME on this host (bench.py's CPU arm): the
    x86-64-v4 (AVX-512) build when the host has AVX-512 -- the nearest
    portable equivalent of the reference's -march=native -- else the v3 one."""
    if os.path.exists(REF_SO_V4) and host_has_avx512():
        return REF_SO_V4, "-O3 -march=x86-64-v4 (AVX-512; host has avx512f/bw/cd/dq/vl)"
    return REF_SO, "-O3 -march=x86-64-v3 (AVX2+FMA)"
