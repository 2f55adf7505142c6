"""TEST INFRASTRUCTURE — ctypes access to the two CPU oracles.

``restatement()`` -> oracle/_build/libfsoracle.so (plain-C restatement, fso_*)
``reference()``   -> oracle/_ref/libfsref.so (the reference compiled from
                     /root/reference by oracle/Makefile, fsref_*)
Both expose the same signatures (oracle/fs_oracle.h) and are wrapped here in
one numpy-level class with the same method names as the product's Python API.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "_build", "libfsoracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libfsref.so")

P, I, D = C.c_void_p, C.c_int, C.c_double
_SIGS = {
    "to_gray": (I, [P, I, I, I, P]),
    "bilinear_sample": (None, [P, P, I, I, I, D, D, P]),
    "compute_partition": (I, [P, P, I, I, P, P]),
    "crop_overlap": (I, [P, P, I, I, I, P, P, P, P, P]),
    "place_on_canvas": (I, [P, P, I, I, I, I, I, I, I, P, P]),
    "build_pyramid": (I, [P, I, I, I, P]),
    "dense_pyr_lk": (I, [P, P, I, I, I, I, I, D, I, P, P]),
    "bidirectional_flow": (I, [P, P, I, I, I, I, I, I, D, I, P, P, P, P]),
    "embed_flow": (I, [P, P, I, I, I, I, I, I, P, P]),
    "flow_magnitude": (None, [P, I, I, P]),
    "distance_transform": (I, [P, I, I, P]),
    "compute_blend": (I, [P, P, I, I, P]),
    "softmax_weights": (None, [D, D, D, D, D, D, P]),
    "blend_pair": (I, [P, P, P, P, I, I, I, P, P, P, P, D, D, P, P]),
    "feather_blend": (I, [P, P, I, I, I, P, P, P, P]),
    "warp_constituents": (I, [P, P, P, P, I, I, I, P, P, P, P, P, P, P, P]),
    "stitch_placed": (I, [I, P, P, P, P, I, I, I, I, I, I, D, I, D, D, P, P]),
    "misalignment_score": (I, [P, P, P, P, I, I, I, P, P, I, I, P]),
    "estimate_translation": (I, [P, P, I, I, I, I, P, P, P]),
}


class OracleError(RuntimeError):
    def __init__(self, status: int, what: str):
        super().__init__(f"{what}: oracle status {status}")
        self.status = status


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _flow_args(params):
    if params is None:
        return (4, 8, 3, 1e-4, 2)
    if hasattr(params, "astuple"):
        return params.astuple()
    return tuple(params)


class Oracle:
    def __init__(self, path: str, prefix: str):
        self.path = path
        self.lib = C.CDLL(path)
        self.prefix = prefix
        for name, (res, args) in _SIGS.items():
            fn = getattr(self.lib, prefix + name)
            fn.restype = res
            fn.argtypes = args
        if prefix == "fsref_":
            self.lib.fsref_set_threads.argtypes = [I]
            self.lib.fsref_resolved_threads.restype = I
            self.lib.fsref_stitch_placed_timed.restype = I
            self.lib.fsref_stitch_placed_timed.argtypes = _SIGS["stitch_placed"][1] + [P]
            self.lib.fsref_stitch_placed_flows.restype = I
            self.lib.fsref_stitch_placed_flows.argtypes = _SIGS["stitch_placed"][1] + [P, P, P]
            self.lib.fsref_stitch_placed_full.restype = I
            self.lib.fsref_stitch_placed_full.argtypes = _SIGS["stitch_placed"][1]

    def _fn(self, name):
        return getattr(self.lib, self.prefix + name)

    def _ok(self, st, what):
        if st != 0:
            raise OracleError(st, what)

    def set_threads(self, n: int):
        if self.prefix == "fsref_":
            self.lib.fsref_set_threads(int(n))

    def threads(self) -> int:
        return self.lib.fsref_resolved_threads() if self.prefix == "fsref_" else 1

    # ---- imagecore ----
    def to_gray(self, data: np.ndarray) -> np.ndarray:
        data = np.ascontiguousarray(data, np.float32)
        h, w, ch = data.shape
        out = np.empty((h, w), np.float32)
        self._ok(self._fn("to_gray")(_p(data), w, h, ch, _p(out)), "to_gray")
        return out

    def bilinear_sample(self, data, valid, x, y) -> np.ndarray:
        data = np.ascontiguousarray(data, np.float32)
        h, w, ch = data.shape
        out = np.empty(ch, np.float32)
        self._fn("bilinear_sample")(_p(data), _p(np.ascontiguousarray(valid, np.uint8)), w, h, ch,
                                    float(x), float(y), _p(out))
        return out

    def compute_partition(self, ml, mr):
        ml = np.ascontiguousarray(ml, np.uint8)
        mr = np.ascontiguousarray(mr, np.uint8)
        h, w = ml.shape
        label = np.empty((h, w), np.uint8)
        counts = np.zeros(4, np.int64)
        self._ok(self._fn("compute_partition")(_p(ml), _p(mr), w, h, _p(label), _p(counts)),
                 "compute_partition")
        return label, counts

    def crop_overlap(self, data, valid, label, counts):
        data = np.ascontiguousarray(data, np.float32)
        h, w, ch = data.shape
        box = np.zeros(4, np.int32)
        valid = np.ascontiguousarray(valid, np.uint8)
        label = np.ascontiguousarray(label, np.uint8)
        counts = np.ascontiguousarray(counts, np.int64)
        self._ok(self._fn("crop_overlap")(_p(data), _p(valid), w, h, ch, _p(label), _p(counts),
                                          None, None, _p(box)), "crop_overlap")
        out = np.empty((box[3], box[2], ch), np.float32)
        ov = np.empty((box[3], box[2]), np.uint8)
        self._ok(self._fn("crop_overlap")(_p(data), _p(valid), w, h, ch, _p(label), _p(counts),
                                          _p(out), _p(ov), _p(box)), "crop_overlap")
        return out, ov, (int(box[0]), int(box[1]))

    def place_on_canvas(self, data, valid, ox, oy, cw, chh):
        data = np.ascontiguousarray(data, np.float32)
        h, w, ch = data.shape
        out = np.empty((chh, cw, ch), np.float32)
        ov = np.empty((chh, cw), np.uint8)
        self._ok(self._fn("place_on_canvas")(_p(data), _p(np.ascontiguousarray(valid, np.uint8)),
                                             w, h, ch, ox, oy, cw, chh, _p(out), _p(ov)),
                 "place_on_canvas")
        return out, ov

    # ---- optflow ----
    def build_pyramid(self, gray: np.ndarray, levels: int) -> List[np.ndarray]:
        gray = np.ascontiguousarray(gray, np.float32)
        h, w = gray.shape
        out = np.empty(w * h * 2 + 64, np.float32)
        depth = self._fn("build_pyramid")(_p(gray), w, h, levels, _p(out))
        if depth <= 0:
            raise OracleError(-depth, "build_pyramid")
        res, off = [], 0
        for _ in range(depth):
            res.append(out[off:off + w * h].reshape(h, w).copy())
            off += w * h
            w, h = max(1, w // 2), max(1, h // 2)
        return res

    def dense_pyr_lk(self, frm, to, params=None):
        frm = np.ascontiguousarray(frm, np.float32)
        to = np.ascontiguousarray(to, np.float32)
        h, w = frm.shape[:2]
        vec = np.empty((h, w, 2), np.float32)
        valid = np.empty((h, w), np.uint8)
        self._ok(self._fn("dense_pyr_lk")(_p(frm), _p(to), w, h, *_flow_args(params), _p(vec),
                                          _p(valid)), "dense_pyr_lk")
        return vec, valid

    def bidirectional_flow(self, l, r, params=None):
        l = np.ascontiguousarray(l, np.float32)
        r = np.ascontiguousarray(r, np.float32)
        if l.ndim == 2:
            l, r = l[:, :, None], r[:, :, None]
        h, w, ch = l.shape
        out = [np.empty((h, w, 2), np.float32), np.empty((h, w), np.uint8),
               np.empty((h, w, 2), np.float32), np.empty((h, w), np.uint8)]
        self._ok(self._fn("bidirectional_flow")(_p(l), _p(r), w, h, ch, *_flow_args(params),
                                                *[_p(o) for o in out]), "bidirectional_flow")
        return (out[0], out[1]), (out[2], out[3])

    def embed_flow(self, vec, valid, ox, oy, cw, chh):
        vec = np.ascontiguousarray(vec, np.float32)
        h, w = vec.shape[:2]
        ov = np.empty((chh, cw, 2), np.float32)
        oval = np.empty((chh, cw), np.uint8)
        self._ok(self._fn("embed_flow")(_p(vec), _p(np.ascontiguousarray(valid, np.uint8)), w, h,
                                        ox, oy, cw, chh, _p(ov), _p(oval)), "embed_flow")
        return ov, oval

    def flow_magnitude(self, vec):
        vec = np.ascontiguousarray(vec, np.float32)
        h, w = vec.shape[:2]
        out = np.empty((h, w), np.float32)
        self._fn("flow_magnitude")(_p(vec), w, h, _p(out))
        return out

    # ---- blend field / blender ----
    def distance_transform(self, mask):
        mask = np.ascontiguousarray(mask, np.uint8)
        h, w = mask.shape
        out = np.empty((h, w), np.float64)
        self._ok(self._fn("distance_transform")(_p(mask), w, h, _p(out)), "distance_transform")
        return out

    def compute_blend(self, label, counts):
        label = np.ascontiguousarray(label, np.uint8)
        h, w = label.shape
        out = np.empty((h, w), np.float64)
        self._ok(self._fn("compute_blend")(_p(label), _p(np.ascontiguousarray(counts, np.int64)),
                                           w, h, _p(out)), "compute_blend")
        return out

    def misalignment_score(self, L, vL, R, vR, label, counts, patch_radius=8, stride=32):
        """proj/src/pipeline.cpp:309-396 -> float score."""
        L = np.ascontiguousarray(L, np.float32)
        R = np.ascontiguousarray(R, np.float32)
        h, w = L.shape[:2]
        ch = 1 if L.ndim == 2 else L.shape[2]
        out = np.zeros(1, np.float64)
        vL = None if vL is None else np.ascontiguousarray(vL, np.uint8)
        self._ok(self._fn("misalignment_score")(
            _p(L), _p(vL), _p(R), _p(np.ascontiguousarray(vR, np.uint8)), w, h, ch,
            _p(np.ascontiguousarray(label, np.uint8)), _p(np.ascontiguousarray(counts, np.int64)),
            patch_radius, stride, _p(out)), "misalignment_score")
        return float(out[0])

    def estimate_translation(self, A, B, max_shift):
        """proj/src/pipeline.cpp:261-307 -> (dx, dy, score)."""
        A = np.ascontiguousarray(A, np.float32)
        B = np.ascontiguousarray(B, np.float32)
        h, w = A.shape[:2]
        ch = 1 if A.ndim == 2 else A.shape[2]
        dx, dy, sc = C.c_int(), C.c_int(), C.c_double()
        self._ok(self._fn("estimate_translation")(_p(A), _p(B), w, h, ch, max_shift, C.byref(dx),
                                                  C.byref(dy), C.byref(sc)), "estimate_translation")
        return dx.value, dy.value, sc.value

    def softmax_weights(self, bl, br, mrl, mlr, k=10.0, coef=0.05):
        out = np.empty(2, np.float64)
        self._fn("softmax_weights")(bl, br, mrl, mlr, k, coef, _p(out))
        return float(out[0]), float(out[1])

    def blend_pair(self, L, vL, R, vR, flow_lr, flow_rl, b, label, k=10.0, coef=0.05):
        L = np.ascontiguousarray(L, np.float32)
        h, w, ch = L.shape
        out = np.empty_like(L)
        ov = np.empty((h, w), np.uint8)
        self._ok(self._fn("blend_pair")(
            _p(L), _p(np.ascontiguousarray(vL, np.uint8)), _p(np.ascontiguousarray(R, np.float32)),
            _p(np.ascontiguousarray(vR, np.uint8)), w, h, ch,
            _p(np.ascontiguousarray(flow_lr, np.float32)),
            _p(np.ascontiguousarray(flow_rl, np.float32)), _p(np.ascontiguousarray(b, np.float64)),
            _p(np.ascontiguousarray(label, np.uint8)), k, coef, _p(out), _p(ov)), "blend_pair")
        return out, ov

    def feather_blend(self, L, R, b, label):
        L = np.ascontiguousarray(L, np.float32)
        h, w, ch = L.shape
        out = np.empty_like(L)
        ov = np.empty((h, w), np.uint8)
        self._ok(self._fn("feather_blend")(
            _p(L), _p(np.ascontiguousarray(R, np.float32)), w, h, ch,
            _p(np.ascontiguousarray(b, np.float64)), _p(np.ascontiguousarray(label, np.uint8)),
            _p(out), _p(ov)), "feather_blend")
        return out, ov

    def warp_constituents(self, L, vL, R, vR, flow_lr, flow_rl, b, label):
        L = np.ascontiguousarray(L, np.float32)
        h, w, ch = L.shape
        ol, orr = np.empty_like(L), np.empty_like(L)
        vl, vr = np.empty((h, w), np.uint8), np.empty((h, w), np.uint8)
        self._ok(self._fn("warp_constituents")(
            _p(L), _p(np.ascontiguousarray(vL, np.uint8)), _p(np.ascontiguousarray(R, np.float32)),
            _p(np.ascontiguousarray(vR, np.uint8)), w, h, ch,
            _p(np.ascontiguousarray(flow_lr, np.float32)),
            _p(np.ascontiguousarray(flow_rl, np.float32)), _p(np.ascontiguousarray(b, np.float64)),
            _p(np.ascontiguousarray(label, np.uint8)), _p(ol), _p(vl), _p(orr), _p(vr)),
            "warp_constituents")
        return (ol, vl), (orr, vr)

    # ---- fold ----
    def _stitch_args(self, images, valids, offsets, cw, chh, params, k, coef):
        n = len(images)
        images = [np.ascontiguousarray(im, np.float32) for im in images]
        valids = [np.ascontiguousarray(v, np.uint8) for v in valids]
        ch = images[0].shape[2]
        imgs = (C.c_void_p * n)(*[im.ctypes.data for im in images])
        vals = (C.c_void_p * n)(*[v.ctypes.data for v in valids])
        dims = np.array([[im.shape[1], im.shape[0]] for im in images], np.int32).ravel()
        offs = np.array(offsets, np.int32).ravel()
        out = np.empty((chh, cw, ch), np.float32)
        ov = np.empty((chh, cw), np.uint8)
        keep = (images, valids, imgs, vals, dims, offs)
        args = [n, C.cast(imgs, C.c_void_p), C.cast(vals, C.c_void_p), _p(dims), _p(offs), ch, cw,
                chh, *_flow_args(params), k, coef, _p(out), _p(ov)]
        return args, out, ov, keep

    def stitch_placed(self, images, valids, offsets, cw, chh, params=None, k=10.0, coef=0.05,
                      timing: Optional[np.ndarray] = None, full=False):
        args, out, ov, keep = self._stitch_args(images, valids, offsets, cw, chh, params, k, coef)
        if timing is not None and self.prefix == "fsref_":
            st = self.lib.fsref_stitch_placed_timed(*args, _p(timing))
        elif full and self.prefix == "fsref_":
            st = self.lib.fsref_stitch_placed_full(*args)
        else:
            st = self._fn("stitch_placed")(*args)
        self._ok(st, "stitch_placed")
        return out, ov

    def stitch_placed_flows(self, images, valids, offsets, cw, chh, params=None, k=10.0,
                            coef=0.05, flows=True):
        """The compiled reference's fold with every fold's crop flows.
        Returns (pano, valid, folds, seconds): folds[k-1] = dict(box=(x, y, w, h),
        lr=(vec, valid), rl=(vec, valid)); seconds = the whole fold's time on
        the host, flow export excluded."""
        if self.prefix != "fsref_":
            raise NotImplementedError("per-fold flows come from the compiled reference")
        args, out, ov, keep = self._stitch_args(images, valids, offsets, cw, chh, params, k, coef)
        folds = []
        CB = C.CFUNCTYPE(None, I, I, I, I, I, P, P, P, P, P)

        def cb(kk, ox, oy, w, h, lr, lrv, rl, rlv, ctx):
            def arr(ptr, shape, dt):
                n = int(np.prod(shape)) * np.dtype(dt).itemsize
                return np.frombuffer(C.string_at(ptr, n), dt).reshape(shape).copy()
            folds.append({"k": kk, "box": (ox, oy, w, h),
                          "lr": (arr(lr, (h, w, 2), np.float32), arr(lrv, (h, w), np.uint8)),
                          "rl": (arr(rl, (h, w, 2), np.float32), arr(rlv, (h, w), np.uint8))})
        cbf = CB(cb)
        timing = np.zeros(6, np.float64)
        st = self.lib.fsref_stitch_placed_flows(*args, _p(timing),
                                                C.cast(cbf, C.c_void_p) if flows else None, None)
        self._ok(st, "stitch_placed_flows")
        return out, ov, folds, float(timing[5])

    def last_report_misalignment(self, max_pairs: int = 64) -> np.ndarray:
        """(before, after) per pair of the last stitch_placed(full=True)
        report of the compiled reference; NaN where the optional is empty."""
        buf = np.full((max_pairs, 2), np.nan)
        fn = self.lib.fsref_last_report_misalignment
        fn.restype = I
        fn.argtypes = [P, I]
        n = fn(_p(buf), max_pairs)
        return buf[:n]


_cache = {}


def restatement() -> Oracle:
    if "fso" not in _cache:
        if not os.path.exists(RESTATEMENT_SO):
            raise FileNotFoundError(f"{RESTATEMENT_SO} not built (make -C oracle)")
        _cache["fso"] = Oracle(RESTATEMENT_SO, "fso_")
    return _cache["fso"]


def ref_available() -> bool:
    return os.path.exists(REFERENCE_SO)


def reference() -> Oracle:
    if "ref" not in _cache:
        if not ref_available():
            raise FileNotFoundError(f"{REFERENCE_SO} not built (make -C oracle with /root/reference)")
        _cache["ref"] = Oracle(REFERENCE_SO, "fsref_")
    return _cache["ref"]
