"""ctypes loaders for the parity checkers -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
arm may import this module.  The product package never does.

* ``Oracle``    -- oracle/build/libcv_oracle.so, our C restatement
                   (oracle/cv_oracle.c) of the reference search.
* ``Reference`` -- oracle/_ref/libcolorvibe_ref_v{3,4}.so, the reference's own
                   src/color.cpp + src/search.cpp behind oracle/ref_shim.cpp.
* ``RefCodec``  -- oracle/_ref/libcolorvibe_ref_codec.so, the reference's own
                   src/codec.cpp (+ search/color/util) behind
                   oracle/ref_codec_shim.cpp.

Both return searches as (idx uint32[n], codes uint8[n, 6], deltas f64[n, 3]),
idx = k * n_angles + m in canonical (radius, angle) order (search.cpp:448-455).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))

_dp = C.POINTER(C.c_double)
_ip = C.POINTER(C.c_int32)
_up = C.POINTER(C.c_uint32)
_bp = C.POINTER(C.c_uint8)
_u64p = C.POINTER(C.c_uint64)


def build() -> None:
    """Runs oracle/Makefile (reference targets skipped when sources absent)."""
    subprocess.run(["make", "-s", "-C", HERE], check=True)


def _cpu_has_avx512() -> bool:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return " avx512f " in line + " "
    except OSError:
        pass
    return False


def _cpu_flags() -> set:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("flags"):
                    return set(line.split(":", 1)[1].split())
    except OSError:
        pass
    return set()


def reference_library() -> str:
    """Path of the reference build for this host: the -march=native build
    (BASELINE.md section 3's flags) when this CPU has every flag of the host
    it was built on (_ref/native_cpu_flags.txt), else x86-64-v4 / -v3."""
    native = os.path.join(HERE, "_ref", "libcolorvibe_ref_native.so")
    flags_file = os.path.join(HERE, "_ref", "native_cpu_flags.txt")
    if os.path.exists(native) and os.path.exists(flags_file):
        with open(flags_file) as f:
            built = set(f.readline().split())
        if built and built <= _cpu_flags():
            return native
    v = "v4" if _cpu_has_avx512() else "v3"
    return os.path.join(HERE, "_ref", f"libcolorvibe_ref_{v}.so")


def _ptr(a, t):
    return None if a is None else a.ctypes.data_as(t)


class _Lib:
    prefix = ""

    def __init__(self, path: str):
        if not os.path.exists(path):
            raise FileNotFoundError(f"parity checker not built: {path} (run oracle/Makefile)")
        self.path = path
        self.lib = C.CDLL(path)
        p = self.prefix
        f = getattr(self.lib, p + "search")
        f.restype = C.c_int64
        f.argtypes = [_ip, C.c_int, C.c_double, C.c_double, _dp, C.c_int, _dp, C.c_int,
                      C.c_int, C.c_int, _dp, C.c_int, C.c_int, _up, _bp, _dp, C.c_int64]
        self._search = f
        for name in ("thresholds", "xyz_to_rgb", "white"):
            getattr(self.lib, p + name).restype = None
        getattr(self.lib, p + "table_code").restype = C.c_int
        getattr(self.lib, p + "table_code").argtypes = [C.c_double]
        getattr(self.lib, p + "quantize").restype = C.c_int
        getattr(self.lib, p + "quantize").argtypes = [C.c_double]

    # -- known-answer constants ------------------------------------------
    def thresholds(self) -> np.ndarray:
        out = np.zeros(256, np.float64)
        getattr(self.lib, self.prefix + "thresholds")(_ptr(out, _dp))
        return out

    def xyz_to_rgb(self) -> np.ndarray:
        out = np.zeros(9, np.float64)
        getattr(self.lib, self.prefix + "xyz_to_rgb")(_ptr(out, _dp))
        return out.reshape(3, 3)

    def white(self) -> np.ndarray:
        out = np.zeros(3, np.float64)
        getattr(self.lib, self.prefix + "white")(_ptr(out, _dp))
        return out

    def table_code(self, x: float) -> int:
        return getattr(self.lib, self.prefix + "table_code")(float(x))

    def quantize(self, x: float) -> int:
        return getattr(self.lib, self.prefix + "quantize")(float(x))

    def srgb_to_lab(self, rgb) -> np.ndarray:
        t = np.ascontiguousarray(rgb, np.int32)
        out = np.zeros(3, np.float64)
        getattr(self.lib, self.prefix + "srgb_to_lab")(*self._lab_args(t, out))
        return out

    def _lab_args(self, t, out):
        return (_ptr(t, _ip), _ptr(out, _dp))

    # -- one search ----------------------------------------------------------
    def search(self, rgb, pattern_bits: int, v_th: float, r_novib: float, radii, angles,
               delta_mode: int = 0, delta_basis: int = 0, white=None, method: int = 1,
               workers: int = 1, want_deltas: bool = True):
        t = np.ascontiguousarray(rgb, np.int32)
        r = np.ascontiguousarray(radii, np.float64)
        a = np.ascontiguousarray(angles, np.float64)
        wp = None if white is None else np.ascontiguousarray(white, np.float64)
        args = [_ptr(t, _ip), int(pattern_bits), float(v_th), float(r_novib),
                _ptr(r, _dp), len(r), _ptr(a, _dp), len(a), int(delta_mode),
                int(delta_basis), _ptr(wp, _dp), int(method), int(workers)]
        n = self._search(*args, None, None, None, 0)
        if n < 0:
            raise ValueError(self.last_error())
        idx = np.zeros(n, np.uint32)
        codes = np.zeros((n, 6), np.uint8)
        deltas = np.zeros((n, 3), np.float64) if want_deltas else None
        if n:
            n2 = self._search(*args, _ptr(idx, _up), _ptr(codes, _bp),
                              _ptr(deltas, _dp), n)
            assert n2 == n
        return idx, codes, deltas

    def last_error(self) -> str:
        return "invalid argument"


class Oracle(_Lib):
    prefix = "cvo_"

    def __init__(self, path: str | None = None):
        super().__init__(path or os.path.join(HERE, "build", "libcv_oracle.so"))
        self.lib.cvo_srgb_to_lab.argtypes = [_ip, _dp, _dp]
        self.lib.cvo_lab_to_linear.argtypes = [_dp, _dp, _dp]

    def _lab_args(self, t, out):
        return (_ptr(t, _ip), None, _ptr(out, _dp))

    def lab_to_linear(self, lab, white=None) -> np.ndarray:
        l = np.ascontiguousarray(lab, np.float64)
        out = np.zeros(3, np.float64)
        wp = None if white is None else np.ascontiguousarray(white, np.float64)
        self.lib.cvo_lab_to_linear(_ptr(l, _dp), _ptr(wp, _dp), _ptr(out, _dp))
        return out


class Reference(_Lib):
    prefix = "cvr_"

    def __init__(self, path: str | None = None):
        super().__init__(path or reference_library())
        self.lib.cvr_last_error.restype = C.c_char_p
        self.lib.cvr_srgb_to_lab.argtypes = [_ip, _dp]
        f = self.lib.cvr_search_many
        f.restype = C.c_int64
        f.argtypes = [C.c_int, _ip, _ip, _dp, _dp, _dp, C.c_int, _dp, C.c_int, C.c_int, _u64p]
        f = self.lib.cvr_search_memo
        f.restype = C.c_int64
        f.argtypes = [C.c_int64, _ip, C.c_int, C.c_double, C.c_double, _dp, C.c_int, _dp, C.c_int, C.c_int,
                      C.c_int, _u64p, _up, _bp]
        self.lib.cvr_batch_search_addr.restype = C.c_void_p

    def batch_search_addr(self) -> int:
        """Address colorvibe::batch_search resolves to inside this library."""
        return self.lib.cvr_batch_search_addr()

    def search_memo(self, rgb, pattern_bits: int, v_th: float, r_novib: float, radii, angles, threads: int = 0,
                    memo: bool = True):
        """Per-pixel batch on an outer pool of `threads` (reference
        batch_search with workers = 1 per pixel), memoized by color
         unless memo=False:
        (counts u64[n], first_idx u32[n], first_codes u8[n, 6], n_searched)."""
        t = np.ascontiguousarray(rgb, np.int32).reshape(-1, 3)
        r = np.ascontiguousarray(radii, np.float64)
        a = np.ascontiguousarray(angles, np.float64)
        n = len(t)
        counts = np.zeros(n, np.uint64)
        first = np.zeros(n, np.uint32)
        codes = np.zeros((n, 6), np.uint8)
        u = self.lib.cvr_search_memo(n, _ptr(t, _ip), int(pattern_bits), float(v_th), float(r_novib),
                                     _ptr(r, _dp), len(r), _ptr(a, _dp), len(a), int(threads or os.cpu_count() or 1),
                                     int(bool(memo)), _ptr(counts, _u64p), _ptr(first, _up), _ptr(codes, _bp))
        if u < 0:
            raise ValueError(self.last_error())
        return counts, first, codes, int(u)

    def last_error(self) -> str:
        return self.lib.cvr_last_error().decode()

    def search_many(self, rgb, patterns, v_th, r_novib, radii, angles, workers: int = 0):
        """Reference batch_search once per search (feasibility.cpp:273-275); counts only."""
        t = np.ascontiguousarray(rgb, np.int32).reshape(-1, 3)
        p = np.ascontiguousarray(patterns, np.int32)
        v = np.ascontiguousarray(v_th, np.float64)
        q = np.ascontiguousarray(r_novib, np.float64)
        r = np.ascontiguousarray(radii, np.float64)
        a = np.ascontiguousarray(angles, np.float64)
        counts = np.zeros(len(t), np.uint64)
        n = self.lib.cvr_search_many(len(t), _ptr(t, _ip), _ptr(p, _ip), _ptr(v, _dp),
                                     _ptr(q, _dp), _ptr(r, _dp), len(r), _ptr(a, _dp),
                                     len(a), int(workers), _ptr(counts, _u64p))
        if n < 0:
            raise ValueError(self.last_error())
        return counts


class RefCodec:
    """The reference codec (codec.cpp) and feasibility sweep (feasibility.cpp)
    through oracle/ref_codec_shim.cpp."""

    def __init__(self, path: str | None = None):
        path = path or os.path.join(HERE, "_ref", "libcolorvibe_ref_codec.so")
        if not os.path.exists(path):
            raise FileNotFoundError(f"reference codec not built: {path} (run oracle/Makefile)")
        self.path = path
        self.lib = C.CDLL(path)
        self.lib.cvrc_last_error.restype = C.c_char_p
        self.lib.cvrc_embed.argtypes = [_bp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _ip, _ip, _ip,
                                        C.POINTER(C.c_char_p), C.c_double, C.c_double, C.c_double, _dp, C.c_int,
                                        _dp, C.c_int, C.c_int, _bp, _bp]
        self.lib.cvrc_decode.argtypes = [_bp, _bp, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                         _ip, _ip, _ip, C.c_double, C.c_double, _ip, _ip, _dp]
        self.lib.cvrc_layout_json.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _ip, C.POINTER(C.c_char_p),
                                              C.c_double, C.c_double, C.c_char_p, C.c_int]
        self.lib.cvrc_report_json.argtypes = [C.c_int, C.c_int, C.c_int, _ip, _ip, _ip, C.POINTER(C.c_char_p),
                                              C.c_double, C.c_double, _ip, _ip, _dp, C.c_char_p, C.c_int]
        self.lib.cvrf_config_roundtrip.argtypes = [C.c_char_p, C.c_char_p, C.c_int, C.c_char_p]
        self.lib.cvrf_export.argtypes = [C.c_char_p, C.c_int, C.c_int, C.c_char_p, C.c_int]

    def config_roundtrip(self, text: str):
        """(config_to_json(config_from_json(text)), config_hash) of the reference."""
        buf, h = C.create_string_buffer(1 << 22), C.create_string_buffer(32)
        n = self.lib.cvrf_config_roundtrip(text.encode(), buf, len(buf), h)
        if n < 0:
            self._raise(-n)
        return buf.value.decode(), h.value.decode()

    def export(self, text: str, fmt: str = "csv", aggregated: bool = True) -> str:
        """export_matrix of the reference's own feasibility_matrix (CPU)."""
        buf = C.create_string_buffer(1 << 24)
        n = self.lib.cvrf_export(text.encode(), int(fmt == "json"), int(aggregated), buf, len(buf))
        if n < 0:
            self._raise(-n)
        return buf.value.decode()

    @staticmethod
    def _layout(xy, rgb, bits, names):
        xy = np.ascontiguousarray(xy, np.int32).reshape(-1, 2)
        rgb = np.ascontiguousarray(rgb, np.int32).reshape(-1, 3)
        bits = np.ascontiguousarray(bits, np.int32).reshape(-1)
        cnames = None
        if names is not None:
            cnames = (C.c_char_p * len(names))(*[n.encode() for n in names])
        return xy, rgb, bits, cnames

    def _raise(self, rc):
        msg = self.lib.cvrc_last_error().decode()
        if rc == 1:
            raise ValueError(msg)
        raise RuntimeError(msg)

    def embed(self, base, bw, bh, xy, rgb, bits, v_th, r_novib, radii, angles, names=None, refresh_hz=60.0,
              basis=0):
        base = np.ascontiguousarray(base, np.uint8)
        h, w = base.shape[:2]
        xy, rgb, bits, cnames = self._layout(xy, rgb, bits, names)
        r = np.ascontiguousarray(radii, np.float64)
        a = np.ascontiguousarray(angles, np.float64)
        fa = np.zeros_like(base)
        fb = np.zeros_like(base)
        rc = self.lib.cvrc_embed(_ptr(base, _bp), w, h, bw, bh, len(xy), _ptr(xy, _ip), _ptr(rgb, _ip),
                                 _ptr(bits, _ip), cnames, v_th, r_novib, refresh_hz, _ptr(r, _dp), len(r),
                                 _ptr(a, _dp), len(a), basis, _ptr(fa, _bp), _ptr(fb, _bp))
        if rc:
            self._raise(rc)
        return fa, fb

    def decode(self, fa, fb, bw, bh, xy, rgb, bits, v_th, r_novib):
        fa = np.ascontiguousarray(fa, np.uint8)
        fb = np.ascontiguousarray(fb, np.uint8)
        xy, rgb, bits, _ = self._layout(xy, rgb, bits, None)
        n = len(xy)
        st = np.zeros(n, np.int32)
        pat = np.zeros(n, np.int32)
        md = np.zeros((n, 3), np.float64)
        rc = self.lib.cvrc_decode(_ptr(fa, _bp), _ptr(fb, _bp), fa.shape[1], fa.shape[0], fb.shape[1], fb.shape[0],
                                  bw, bh, n, _ptr(xy, _ip), _ptr(rgb, _ip), _ptr(bits, _ip), v_th, r_novib,
                                  _ptr(st, _ip), _ptr(pat, _ip), _ptr(md, _dp))
        if rc:
            self._raise(rc)
        return st, pat, md

    def layout_json(self, bw, bh, xy, rgb, bits, names, v_th, r_novib) -> str:
        xy, rgb, bits, cnames = self._layout(xy, rgb, bits, names)
        buf = C.create_string_buffer(1 << 20)
        n = self.lib.cvrc_layout_json(bw, bh, len(xy), _ptr(xy, _ip), _ptr(rgb, _ip), _ptr(bits, _ip), cnames,
                                      v_th, r_novib, buf, len(buf))
        if n < 0:
            self._raise(1)
        return buf.value.decode()

    def report_json(self, bw, bh, xy, rgb, bits, names, v_th, r_novib, status, pattern, mean_deltas) -> str:
        xy, rgb, bits, cnames = self._layout(xy, rgb, bits, names)
        st = np.ascontiguousarray(status, np.int32)
        pat = np.ascontiguousarray(pattern, np.int32)
        md = np.ascontiguousarray(mean_deltas, np.float64)
        buf = C.create_string_buffer(1 << 20)
        n = self.lib.cvrc_report_json(bw, bh, len(xy), _ptr(xy, _ip), _ptr(rgb, _ip), _ptr(bits, _ip), cnames,
                                      v_th, r_novib, _ptr(st, _ip), _ptr(pat, _ip), _ptr(md, _dp), buf, len(buf))
        if n < 0:
            self._raise(1)
        return buf.value.decode()
