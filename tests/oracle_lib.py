"""ctypes bindings for the TEST-ONLY checkers under oracle/.

- ``Oracle``: the C restatement (oracle/liboracle.so), available everywhere the
  repo is built (it travels to the GPU box in-tree).
- ``Reference``: the unmodified reference sources compiled in place
  (oracle/_ref/libbandmatch_ref.so).  Built by ``make -C oracle`` where
  /root/reference exists; the prebuilt .so also travels to the GPU box.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg may use
this module, and only as the checker / the timed CPU baseline.
"""
from __future__ import annotations

import ctypes as C
import os
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "liboracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libbandmatch_ref.so"

DIM = 128
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C")
_u32p = np.ctypeslib.ndpointer(np.uint32, flags="C")
_u64p = np.ctypeslib.ndpointer(np.uint64, flags="C")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C")


class HashParams(C.Structure):
    _fields_ = [("tables", C.c_int32), ("coarse_bits", C.c_int32), ("fine_bits", C.c_int32)]


def fine_words(fine_bits: int) -> int:
    return (fine_bits + 63) // 64


def _arr(a, dt):
    return np.ascontiguousarray(a, dtype=dt)


class Oracle:
    """C restatement of hashmatch.cpp / engine.cpp row body."""

    def __init__(self, path: Path = ORACLE_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = C.CDLL(str(path))
        L.orc_seed_for.restype = C.c_uint64
        L.orc_seed_for.argtypes = [C.c_uint64, C.c_char_p]
        L.orc_make_hash_functions.argtypes = [C.c_uint64, C.POINTER(HashParams), _f32p, _f32p]
        L.orc_row_mean.argtypes = [C.POINTER(C.c_void_p), _u64p, C.c_size_t, _f32p]
        L.orc_row_mean.restype = None
        L.orc_compute_codes.argtypes = [_f32p, C.c_uint64, C.POINTER(HashParams), _f32p, _f32p,
                                        _f32p, _u32p, _u64p]
        L.orc_centered_dot.restype = C.c_double
        L.orc_centered_dot.argtypes = [_f32p, _f32p, _f32p]
        L.orc_euclidean.restype = C.c_double
        L.orc_euclidean.argtypes = [_f32p, _f32p]
        L.orc_match_pair.argtypes = [_f32p, C.c_uint64, _u32p, _u64p, _f32p, C.c_uint64, _u32p,
                                     _u64p, C.POINTER(HashParams), C.c_int32, C.c_double, _i32p,
                                     C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p]
        L.orc_brute_force_match.argtypes = [_f32p, C.c_uint64, _f32p, C.c_uint64, C.c_double,
                                            _i32p, C.POINTER(C.c_uint64)]

    def seed_for(self, root: int, tag: str) -> int:
        return self.lib.orc_seed_for(root, tag.encode())

    def make_hash_functions(self, seed, tables=6, coarse_bits=8, fine_bits=128):
        hp = HashParams(tables, coarse_bits, fine_bits)
        coarse = np.zeros(max(tables * coarse_bits, 0) * DIM, np.float32)
        fine = np.zeros(max(fine_bits, 0) * DIM, np.float32)
        rc = self.lib.orc_make_hash_functions(seed, C.byref(hp), coarse, fine)
        if rc != 0:
            raise ValueError("InvalidArgument")
        return coarse.reshape(tables, coarse_bits, DIM), fine.reshape(fine_bits, DIM)

    def row_mean(self, images):
        arrs = [_arr(a, np.float32).reshape(-1, DIM) for a in images]
        ptrs = (C.c_void_p * max(1, len(arrs)))(*[a.ctypes.data for a in arrs])
        counts = np.array([a.shape[0] for a in arrs] or [0], np.uint64)
        out = np.zeros(DIM, np.float32)
        self.lib.orc_row_mean(ptrs, counts, len(arrs), out)
        return out

    def compute_codes(self, desc, coarse, fine, mean):
        desc = _arr(desc, np.float32).reshape(-1, DIM)
        tables, cb = coarse.shape[0], coarse.shape[1]
        fb = fine.shape[0]
        hp = HashParams(tables, cb, fb)
        n = desc.shape[0]
        cout = np.zeros(max(n, 1) * tables, np.uint32)
        fout = np.zeros(max(n, 1) * fine_words(fb), np.uint64)
        rc = self.lib.orc_compute_codes(desc, n, C.byref(hp), _arr(coarse, np.float32).ravel(),
                                        _arr(fine, np.float32).ravel(), _arr(mean, np.float32),
                                        cout, fout)
        if rc != 0:
            raise ValueError("InvalidArgument")
        return cout[: n * tables].reshape(n, tables), fout[: n * fine_words(fb)].reshape(n, fine_words(fb))

    def match_pair(self, qdesc, qcodes, tdesc, tcodes, params, k=8, ratio=0.5, diagnostics=False):
        qdesc = _arr(qdesc, np.float32).reshape(-1, DIM)
        tdesc = _arr(tdesc, np.float32).reshape(-1, DIM)
        hp = HashParams(*params)
        nq, nt = qdesc.shape[0], tdesc.shape[0]
        out = np.zeros(2 * max(nq, 1), np.int32)
        cnt = C.c_uint64(0)
        cand = np.zeros(max(nq, 1), np.uint32) if diagnostics else None
        topk = np.zeros(max(nq, 1) * max(k, 1), np.uint64) if diagnostics else None
        rc = self.lib.orc_match_pair(
            qdesc, nq, _arr(qcodes[0], np.uint32).ravel() if nq else np.zeros(1, np.uint32),
            _arr(qcodes[1], np.uint64).ravel() if nq else np.zeros(1, np.uint64), tdesc, nt,
            _arr(tcodes[0], np.uint32).ravel() if nt else np.zeros(1, np.uint32),
            _arr(tcodes[1], np.uint64).ravel() if nt else np.zeros(1, np.uint64), C.byref(hp), k,
            ratio, out, C.byref(cnt), cand.ctypes.data if diagnostics else None,
            topk.ctypes.data if diagnostics else None)
        if rc == 1:
            raise ValueError("InvalidArgument")
        if rc != 0:
            raise RuntimeError(f"oracle match_pair failed rc={rc}")
        m = out[: 2 * cnt.value].reshape(-1, 2)
        if diagnostics:
            return m, cand[:nq], topk[: nq * k].reshape(nq, k)
        return m

    def encode_vlad(self, desc, centroids):
        """encode_vlad (retrieval.cpp:160-205): (values [k*128], degenerate)."""
        c = _arr(centroids, np.float32).reshape(-1, DIM)
        d = _arr(desc, np.float32).reshape(-1, DIM)
        k = len(c)
        out = np.zeros(max(k * DIM, 1), np.float32)
        deg = np.zeros(1, np.uint8)
        self.lib.orc_encode_vlad.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        rc = self.lib.orc_encode_vlad(c.ctypes.data, k, d.ctypes.data, len(d), out.ctypes.data, deg.ctypes.data)
        if rc != 0:
            raise ValueError("InvalidArgument: codebook has no words")
        return out[: k * DIM], bool(deg[0])

    def brute_force_match(self, qdesc, tdesc, ratio=0.5):
        qdesc = _arr(qdesc, np.float32).reshape(-1, DIM)
        tdesc = _arr(tdesc, np.float32).reshape(-1, DIM)
        out = np.zeros(2 * max(qdesc.shape[0], 1), np.int32)
        cnt = C.c_uint64(0)
        self.lib.orc_brute_force_match(qdesc, qdesc.shape[0], tdesc, tdesc.shape[0], ratio, out,
                                       C.byref(cnt))
        return out[: 2 * cnt.value].reshape(-1, 2)


class Reference:
    """The compiled reference library (oracle/_ref)."""

    def __init__(self, path: Path = REF_SO):
        if not path.exists():
            raise FileNotFoundError(f"{path} missing: run `make -C oracle` where /root/reference exists")
        L = self.lib = C.CDLL(str(path))
        L.ref_last_error.restype = C.c_char_p
        L.ref_seed_for.restype = C.c_uint64
        L.ref_seed_for.argtypes = [C.c_uint64, C.c_char_p]
        L.ref_make_hash_functions.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, _f32p, _f32p]
        L.ref_compute_codes.argtypes = [_f32p, C.c_uint64, C.c_uint64, C.c_int, C.c_int, C.c_int,
                                        _f32p, _f32p, _f32p, _u32p, _u64p]
        L.ref_match_pair.argtypes = [_f32p, C.c_uint64, _u32p, _u64p, _f32p, C.c_uint64, _u32p,
                                     _u64p, C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.c_double, _i32p, C.POINTER(C.c_uint64)]
        L.ref_brute_force_match.argtypes = [_f32p, C.c_uint64, _f32p, C.c_uint64, C.c_double,
                                            _i32p, C.POINTER(C.c_uint64)]
        L.ref_synth_create.restype = C.c_void_p
        L.ref_synth_create.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                       C.c_uint64]
        L.ref_synth_count.restype = C.c_uint64
        L.ref_synth_count.argtypes = [C.c_void_p, C.c_int]
        L.ref_synth_copy.argtypes = [C.c_void_p, C.c_int, _f32p]
        L.ref_synth_copy_keypoints.argtypes = [C.c_void_p, C.c_int, _f32p]
        L.ref_synth_pair_count.restype = C.c_uint64
        L.ref_synth_pair_count.argtypes = [C.c_void_p]
        L.ref_synth_pairs.argtypes = [C.c_void_p, _u64p]
        L.ref_synth_free.argtypes = [C.c_void_p]
        L.ref_iterate_schedule_to_file.argtypes = [_u64p, C.c_uint64, _u64p, C.c_uint64, C.c_int,
                                                   C.c_int, C.c_char_p]
        L.ref_features_create.restype = C.c_void_p
        L.ref_features_add.argtypes = [C.c_void_p, C.c_uint64, _f32p, C.c_uint64]
        L.ref_features_free.argtypes = [C.c_void_p]
        L.ref_execute_plan.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int,
                                       C.c_int, C.c_int, C.c_double, C.c_uint64, _u64p, _u64p,
                                       _i32p, C.POINTER(C.c_uint64), C.POINTER(C.c_double), _u64p]
        L.ref_execute_plan_rows.argtypes = [C.c_char_p, C.c_void_p, C.c_uint64, C.c_int, C.c_int,
                                            C.c_int, C.c_int, C.c_double, C.c_int, C.c_uint64,
                                            C.c_uint64, C.POINTER(C.c_uint64),
                                            C.POINTER(C.c_uint64), C.POINTER(C.c_double),
                                            C.POINTER(C.c_void_p)]
        L.ref_results_pairs.restype = C.c_uint64
        L.ref_results_pairs.argtypes = [C.c_void_p]
        L.ref_results_matches.restype = C.c_uint64
        L.ref_results_matches.argtypes = [C.c_void_p]
        L.ref_results_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]
        L.ref_results_free.argtypes = [C.c_void_p]
        L.ref_synth_features.restype = C.c_void_p
        L.ref_synth_features.argtypes = [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double,
                                         C.c_uint64, C.c_int]
        L.ref_features_count.restype = C.c_uint64
        L.ref_features_count.argtypes = [C.c_void_p, C.c_uint64]

        L.ref_knn_from_delaunay.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_void_p,
                                            C.POINTER(C.c_int)]
        L.ref_sao_filter.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                                     C.c_uint64, C.c_int, C.c_double, C.c_void_p, C.c_void_p,
                                     C.POINTER(C.c_uint32)]
        L.ref_write_features.argtypes = [C.c_char_p, C.c_uint64, _f32p, _f32p, C.c_uint64]
        L.ref_read_features.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_uint64),
                                        C.POINTER(C.c_uint64), C.c_void_p, C.c_void_p]
        L.ref_write_matches_binary.argtypes = [C.c_char_p, C.c_uint64, C.c_void_p, C.c_void_p,
                                               C.c_void_p, C.c_void_p]

    def knn_from_delaunay(self, pts, k):
        """knn_from_delaunay (verify.cpp:135-196): (neighbors [n][k] padded
        with -1, used_fallback)."""
        xy = _arr(pts, np.float64).reshape(-1, 2)
        n = len(xy)
        out = np.full(max(n * k, 1), -1, np.int32)
        fb = C.c_int(0)
        self._check(self.lib.ref_knn_from_delaunay(xy.ctypes.data, n, k, out.ctypes.data, C.byref(fb)))
        return out[: n * k].reshape(n, k), bool(fb.value)

    def sao_filter(self, matches, qkp, tkp, n_neighbors=6, threshold=0.5):
        """sao_filter (verify.cpp:303-341): (keep mask, scores, passthrough,
        fallback)."""
        m = _arr(matches, np.int32).reshape(-1, 2)
        qk = _arr(qkp, np.float32).reshape(-1, 4)
        tk = _arr(tkp, np.float32).reshape(-1, 4)
        keep = np.zeros(max(len(m), 1), np.uint8)
        scores = np.zeros(max(len(m), 1), np.float64)
        fl = C.c_uint32(0)
        self._check(self.lib.ref_sao_filter(m.ctypes.data, len(m), qk.ctypes.data, len(qk), tk.ctypes.data,
                                            len(tk), n_neighbors, threshold, keep.ctypes.data,
                                            scores.ctypes.data, C.byref(fl)))
        return keep[: len(m)].astype(bool), scores[: len(m)], bool(fl.value & 1), bool(fl.value & 2)

    def write_features(self, path, image_id, desc, kp):
        desc = _arr(desc, np.float32)
        kp = _arr(kp, np.float32)
        self._check(self.lib.ref_write_features(str(path).encode(), image_id, desc, kp, len(desc)))

    def read_features(self, path):
        """(image_id, descriptors, keypoints) via the reference reader."""
        iid, n = C.c_uint64(0), C.c_uint64(0)
        self._check(self.lib.ref_read_features(str(path).encode(), 0, C.byref(iid), C.byref(n), None, None))
        desc = np.empty((n.value, 128), np.float32)
        kp = np.empty((n.value, 4), np.float32)
        self._check(self.lib.ref_read_features(str(path).encode(), n.value, C.byref(iid), C.byref(n),
                                               desc.ctypes.data, kp.ctypes.data))
        return iid.value, desc, kp

    def write_matches_binary(self, path, pairs, stages=None):
        """pairs: list of (q, t, int32 [m][2]) in any order (the reference sorts)."""
        ids = np.array([(q, t) for q, t, _ in pairs], np.uint64).reshape(-1)
        counts = np.array([len(m) for _, _, m in pairs], np.uint64)
        offs = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
        log = (np.ascontiguousarray(np.concatenate([np.asarray(m, np.int32).reshape(-1, 2) for _, _, m in pairs]))
               if pairs else np.zeros((0, 2), np.int32))
        st = None if stages is None else np.asarray(stages, np.uint8)
        self._check(self.lib.ref_write_matches_binary(str(path).encode(), len(pairs), ids.ctypes.data,
                                                      offs.ctypes.data, log.ctypes.data,
                                                      None if st is None else st.ctypes.data))

    def encode_vlad(self, desc, centroids):
        """the reference encode_vlad: (values [k*128], degenerate)."""
        c = _arr(centroids, np.float32).reshape(-1, DIM)
        d = _arr(desc, np.float32).reshape(-1, DIM)
        k = len(c)
        out = np.zeros(max(k * DIM, 1), np.float32)
        deg = np.zeros(1, np.uint8)
        self.lib.ref_encode_vlad.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p]
        self._check(self.lib.ref_encode_vlad(c.ctypes.data, k, d.ctypes.data, len(d), out.ctypes.data,
                                             deg.ctypes.data))
        return out[: k * DIM], bool(deg[0])

    def encode_vlad_batch(self, images, centroids, threads=1):
        """the reference encode_vlad over images on `threads` host threads:
        (values [n][k*128], degenerate [n])."""
        c = _arr(centroids, np.float32).reshape(-1, DIM)
        arrs = [_arr(x, np.float32).reshape(-1, DIM) for x in images]
        n, k = len(arrs), len(c)
        ptrs = (C.c_void_p * max(n, 1))(*[a.ctypes.data for a in arrs])
        counts = np.array([len(a) for a in arrs] or [0], np.uint64)
        out = np.zeros((max(n, 1), k * DIM), np.float32)
        deg = np.zeros(max(n, 1), np.uint8)
        self.lib.ref_encode_vlad_batch.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_uint64,
                                                   C.c_int, C.c_void_p, C.c_void_p]
        self._check(self.lib.ref_encode_vlad_batch(c.ctypes.data, k, ptrs, counts.ctypes.data, n, threads,
                                                   out.ctypes.data, deg.ctypes.data))
        return out[:n], deg[:n].astype(bool)

    def train_codebook(self, desc, k_words, max_iters=25, seed=0):
        """the reference train_codebook: (centroids [k][128], sse history)."""
        d = _arr(desc, np.float32).reshape(-1, DIM)
        out = np.zeros((k_words, DIM), np.float32)
        sse = np.zeros(max(max_iters, 1), np.float64)
        nse = C.c_int(0)
        self.lib.ref_train_codebook.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_int, C.c_uint64,
                                                C.c_void_p, C.c_void_p, C.POINTER(C.c_int)]
        self._check(self.lib.ref_train_codebook(d.ctypes.data, len(d), k_words, max_iters, seed,
                                                out.ctypes.data, sse.ctypes.data, C.byref(nse)))
        return out, sse[: nse.value]

    def _check(self, rc):
        if rc != 0:
            msg = self.lib.ref_last_error().decode()
            code = msg.split(":")[0]
            raise RefError(code, msg)

    def seed_for(self, root, tag):
        return self.lib.ref_seed_for(root, tag.encode())

    def make_hash_functions(self, seed, tables=6, coarse_bits=8, fine_bits=128):
        coarse = np.zeros(max(tables * coarse_bits, 1) * DIM, np.float32)
        fine = np.zeros(max(fine_bits, 1) * DIM, np.float32)
        self._check(self.lib.ref_make_hash_functions(seed, tables, coarse_bits, fine_bits, coarse,
                                                     fine))
        return (coarse[: tables * coarse_bits * DIM].reshape(tables, coarse_bits, DIM),
                fine[: fine_bits * DIM].reshape(fine_bits, DIM))

    def compute_codes(self, desc, coarse, fine, mean, seed=0):
        desc = _arr(desc, np.float32).reshape(-1, DIM)
        tables, cb, fb = coarse.shape[0], coarse.shape[1], fine.shape[0]
        n = desc.shape[0]
        cout = np.zeros(max(n, 1) * tables, np.uint32)
        fout = np.zeros(max(n, 1) * fine_words(fb), np.uint64)
        self._check(self.lib.ref_compute_codes(
            desc if n else np.zeros(DIM, np.float32), n, seed, tables, cb, fb,
            _arr(coarse, np.float32).ravel(), _arr(fine, np.float32).ravel(),
            _arr(mean, np.float32), cout, fout))
        return cout[: n * tables].reshape(n, tables), fout[: n * fine_words(fb)].reshape(n, fine_words(fb))

    def match_pair(self, qdesc, qcodes, tdesc, tcodes, params, k=8, ratio=0.5, seed=0):
        qdesc = _arr(qdesc, np.float32).reshape(-1, DIM)
        tdesc = _arr(tdesc, np.float32).reshape(-1, DIM)
        nq, nt = qdesc.shape[0], tdesc.shape[0]
        out = np.zeros(2 * max(nq, 1), np.int32)
        cnt = C.c_uint64(0)
        z32, z64, zf = np.zeros(1, np.uint32), np.zeros(1, np.uint64), np.zeros(DIM, np.float32)
        self._check(self.lib.ref_match_pair(
            qdesc if nq else zf, nq, _arr(qcodes[0], np.uint32).ravel() if nq else z32,
            _arr(qcodes[1], np.uint64).ravel() if nq else z64, tdesc if nt else zf, nt,
            _arr(tcodes[0], np.uint32).ravel() if nt else z32,
            _arr(tcodes[1], np.uint64).ravel() if nt else z64, seed, params[0], params[1],
            params[2], k, ratio, out, C.byref(cnt)))
        return out[: 2 * cnt.value].reshape(-1, 2)

    def brute_force_match(self, qdesc, tdesc, ratio=0.5):
        qdesc = _arr(qdesc, np.float32).reshape(-1, DIM)
        tdesc = _arr(tdesc, np.float32).reshape(-1, DIM)
        out = np.zeros(2 * max(qdesc.shape[0], 1), np.int32)
        cnt = C.c_uint64(0)
        self._check(self.lib.ref_brute_force_match(qdesc, qdesc.shape[0], tdesc, tdesc.shape[0],
                                                   ratio, out, C.byref(cnt)))
        return out[: 2 * cnt.value].reshape(-1, 2)

    def generate_synthetic(self, n_images, ppi, band, sigma=0.02, outlier_fraction=0.2, seed=7,
                           keypoints=False):
        h = self.lib.ref_synth_create(n_images, ppi, band, sigma, outlier_fraction, seed)
        if not h:
            self._check(1)
        try:
            images, kps = [], []
            for i in range(n_images):
                n = self.lib.ref_synth_count(h, i)
                a = np.zeros(max(n, 1) * DIM, np.float32)
                self.lib.ref_synth_copy(h, i, a)
                images.append(a[: n * DIM].reshape(n, DIM))
                if keypoints:
                    k = np.zeros(max(n, 1) * 4, np.float32)
                    self.lib.ref_synth_copy_keypoints(h, i, k)
                    kps.append(k[: n * 4].reshape(n, 4))
            np_ = self.lib.ref_synth_pair_count(h)
            pairs = np.zeros(max(np_, 1) * 2, np.uint64)
            self.lib.ref_synth_pairs(h, pairs)
            pairs = pairs[: 2 * np_].reshape(-1, 2)
        finally:
            self.lib.ref_synth_free(h)
        return (images, pairs, kps) if keypoints else (images, pairs)

    def iterate_schedule(self, ids, pairs, size_blk, size_gpu, path):
        ids = np.ascontiguousarray(ids, np.uint64)
        pairs = np.ascontiguousarray(pairs, np.uint64).reshape(-1)
        self._check(self.lib.ref_iterate_schedule_to_file(ids, len(ids), pairs, len(pairs) // 2,
                                                          size_blk, size_gpu, str(path).encode()))

    def _features(self, images):
        h = self.lib.ref_features_create()
        for iid, d in images.items():
            d = _arr(d, np.float32).reshape(-1, DIM)
            self.lib.ref_features_add(h, int(iid), d if len(d) else np.zeros(DIM, np.float32),
                                      len(d))
        return h

    def execute_plan(self, plan_path, images, hash_seed, params=(6, 8, 128), k=8, ratio=0.5,
                     capacity_units=None, max_pairs=100000):
        """Reference execute_plan (verify off).  images: {id: (n,128) f32}."""
        if capacity_units is None:
            capacity_units = 1 << 62
        h = self._features(images)
        try:
            total_q = sum(len(d) for d in images.values())
            pair_ids = np.zeros(2 * max_pairs, np.uint64)
            offsets = np.zeros(max_pairs + 1, np.uint64)
            matches = np.zeros(2 * max(total_q * 64, 1), np.int32)
            npairs, wall = C.c_uint64(0), C.c_double(0)
            counters = np.zeros(6, np.uint64)
            self._check(self.lib.ref_execute_plan(str(plan_path).encode(), h, hash_seed, params[0],
                                                  params[1], params[2], k, ratio, capacity_units,
                                                  pair_ids, offsets, matches, C.byref(npairs),
                                                  C.byref(wall), counters))
        finally:
            self.lib.ref_features_free(h)
        n = npairs.value
        res = {}
        for p in range(n):
            a, b = int(pair_ids[2 * p]), int(pair_ids[2 * p + 1])
            res[(a, b)] = matches[2 * offsets[p]: 2 * offsets[p + 1]].reshape(-1, 2).copy()
        keys = ["pairs_matched", "initial_matches", "uploads", "evictions", "units_uploaded",
                "peak_occupancy"]
        return res, dict(zip(keys, map(int, counters))), wall.value

    def synth_features(self, n_images, ppi, band, sigma=0.02, outlier_fraction=0.2, seed=7, drop=0):
        """The reference generator straight into a reference feature table
        (images [drop, n) renumbered from 0).  Returns a FeatureTable."""
        h = self.lib.ref_synth_features(n_images, ppi, band, sigma, outlier_fraction, seed, drop)
        if not h:
            self._check(1)
        return FeatureTable(self, h, n_images - drop)

    def feature_table(self, images):
        """{id: (n,128) f32} copied into a reference feature table."""
        return FeatureTable(self, self._features(images), len(images))

    def execute_plan_rows(self, plan_path, features, hash_seed, params=(6, 8, 128), k=8, ratio=0.5,
                          threads=None, row_begin=0, row_end=0, want_matches=False):
        """The reference's row body (mean, compute_codes, match_pair) over the
        plan rows [row_begin, row_end) (0 = all) on `threads` threads.
        features: a FeatureTable or {id: array}.  Returns (pairs, matches,
        wall_s, results) with results = (pair_ids [P,2] u64, offsets [P+1]
        u64, matches [M,2] i32) in IdPair order, or None."""
        threads = threads or os.cpu_count()
        own = not isinstance(features, FeatureTable)
        table = self.feature_table(features) if own else features
        res = C.c_void_p(None)
        try:
            done, m, wall = C.c_uint64(0), C.c_uint64(0), C.c_double(0)
            self._check(self.lib.ref_execute_plan_rows(
                str(plan_path).encode(), table.handle, hash_seed, params[0], params[1], params[2], k,
                ratio, threads, row_begin, row_end, C.byref(done), C.byref(m), C.byref(wall),
                C.byref(res) if want_matches else None))
            out = None
            if want_matches and res.value:
                np_ = self.lib.ref_results_pairs(res)
                nm = self.lib.ref_results_matches(res)
                ids = np.zeros((max(np_, 1), 2), np.uint64)
                offs = np.zeros(np_ + 1, np.uint64)
                mt = np.zeros((max(nm, 1), 2), np.int32)
                self.lib.ref_results_copy(res, ids.ctypes.data, offs.ctypes.data, mt.ctypes.data)
                out = (ids[:np_], offs, mt[:nm])
        finally:
            if res.value:
                self.lib.ref_results_free(res)
            if own:
                table.free()
        return done.value, m.value, wall.value, out


class FeatureTable:
    """A std::map<ImageId, FeatureSet> owned by the reference library."""

    def __init__(self, ref, handle, n):
        self.ref, self.handle, self.n = ref, handle, n

    def count(self, image_id):
        return self.ref.lib.ref_features_count(self.handle, image_id)

    def free(self):
        if self.handle:
            self.ref.lib.ref_features_free(self.handle)
            self.handle = None

    def __del__(self):
        self.free()


class RefError(Exception):
    def __init__(self, code, msg):
        super().__init__(msg)
        self.code = code
