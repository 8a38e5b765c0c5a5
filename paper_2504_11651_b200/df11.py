"""Thin Python binding of the C ABI in include/df11.h (argument marshalling only).

Every step of encode and decode runs in libdf11.so (host encoder in C++, decode in sm_100a CUDA
kernels).  PyTorch only provides device memory and the current CUDA stream.  There is no fallback:
if the library is missing the import fails loudly.

Names follow the C ABI: encode / encode_group / decompress / decompress_block / decompress_host.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB_PATH = os.environ.get("DF11_LIB") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "lib",
                                                        "libdf11.so")   # DF11_LIB: A/B builds

DF11_OK = 0
STATUS = {0: "DF11_OK", 1: "DF11_E_INVALID_ARGUMENT", 2: "DF11_E_RESERVED_EXPONENT", 3: "DF11_E_LUT_OVERFLOW",
          4: "DF11_E_TOO_LARGE", 5: "DF11_E_CORRUPT", 6: "DF11_E_CUDA", 7: "DF11_E_ALLOC", 8: "DF11_E_UNSUPPORTED"}
LUT_MODES = {"auto": 0, "narrow": 1, "wide": 2}
# value formats (df11.h DF11_VF_*; NEXT-4): name -> (code, word bytes, residual bits R)
VALUE_FORMATS = {"bf16": (0, 2, 8), "fp16": (1, 2, 11), "fp8_e4m3": (2, 1, 4), "fp8_e5m2": (3, 1, 3)}
VF_NAMES = {v[0]: k for k, v in VALUE_FORMATS.items()}
LUT_BITS_MONOLITHIC = 255
KERNELS = {"auto": 0, "alg1": 1, "fast": 2}
MAX_BATCH = 64

EXPORTED_SYMBOLS = ("df11_encode", "df11_encode_group", "df11_host_tensor_free", "df11_decompress",
                    "df11_decompress_block", "df11_decompress_block_ex", "df11_decompress_block_budget",
                    "df11_decompress_host",
                    "df11_decompress_host_block", "df11_plan_cta_ranges", "df11_status_string", "df11_last_cuda_error", "df11_last_error_message", "df11_version",
                    "df11_launch_count", "df11_last_kernel_mask", "df11_histogram_device", "df11_encode_plan_create",
                    "df11_encode_plan_free", "df11_encode_device")


class Df11Error(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status
        self.kind = STATUS.get(status, str(status))


class EncodeOpts(ctypes.Structure):
    _fields_ = [("threads_per_block", ctypes.c_uint32), ("bytes_per_thread", ctypes.c_uint32),
                ("lut_mode", ctypes.c_uint32), ("num_threads", ctypes.c_uint32),
                ("value_format", ctypes.c_uint32), ("lut_bits", ctypes.c_uint32)]


class HostTensorC(ctypes.Structure):
    _fields_ = [("num_elements", ctypes.c_uint64), ("encoded_bits", ctypes.c_uint64),
                ("T", ctypes.c_uint32), ("n", ctypes.c_uint32), ("B", ctypes.c_uint32), ("k", ctypes.c_uint32),
                ("lut_entry_bytes", ctypes.c_uint32), ("max_code_len", ctypes.c_uint32),
                ("value_format", ctypes.c_uint32), ("lut_bits", ctypes.c_uint32),
                ("code_lengths", ctypes.c_uint8 * 256),
                ("luts", ctypes.POINTER(ctypes.c_uint8)), ("luts_bytes", ctypes.c_uint64),
                ("encoded_exponent", ctypes.POINTER(ctypes.c_uint8)), ("encoded_exponent_bytes", ctypes.c_uint64),
                ("packed_sign_mantissa", ctypes.POINTER(ctypes.c_uint8)),
                ("packed_sign_mantissa_bytes", ctypes.c_uint64),
                ("gaps", ctypes.POINTER(ctypes.c_uint8)), ("gaps_bytes", ctypes.c_uint64),
                ("block_output_pos", ctypes.POINTER(ctypes.c_uint32))]


class DeviceTensorC(ctypes.Structure):
    _fields_ = [("encoded_exponent", ctypes.c_void_p), ("packed_sign_mantissa", ctypes.c_void_p),
                ("gaps", ctypes.c_void_p), ("luts", ctypes.c_void_p), ("code_lengths", ctypes.c_void_p),
                ("block_output_pos", ctypes.c_void_p), ("out", ctypes.c_void_p),
                ("num_elements", ctypes.c_uint64), ("T", ctypes.c_uint32), ("n", ctypes.c_uint32),
                ("B", ctypes.c_uint32), ("k", ctypes.c_uint32), ("lut_entry_bytes", ctypes.c_uint32),
                ("value_format", ctypes.c_uint32), ("lut_bits", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class EncodePlanC(ctypes.Structure):
    _fields_ = [("num_elements", ctypes.c_uint64), ("encoded_bits", ctypes.c_uint64),
                ("T", ctypes.c_uint32), ("n", ctypes.c_uint32), ("B", ctypes.c_uint32), ("k", ctypes.c_uint32),
                ("lut_entry_bytes", ctypes.c_uint32), ("max_code_len", ctypes.c_uint32),
                ("lut_bits", ctypes.c_uint32), ("value_format", ctypes.c_uint32),
                ("code_lengths", ctypes.c_uint8 * 256), ("codes", ctypes.c_uint32 * 256),
                ("luts", ctypes.POINTER(ctypes.c_uint8)), ("luts_bytes", ctypes.c_uint64),
                ("encoded_exponent_bytes", ctypes.c_uint64), ("packed_sign_mantissa_bytes", ctypes.c_uint64),
                ("gaps_bytes", ctypes.c_uint64), ("workspace_bytes", ctypes.c_uint64)]


class DeviceBuffersC(ctypes.Structure):
    _fields_ = [("encoded_exponent", ctypes.c_void_p), ("packed_sign_mantissa", ctypes.c_void_p),
                ("gaps", ctypes.c_void_p), ("luts", ctypes.c_void_p), ("code_lengths", ctypes.c_void_p),
                ("block_output_pos", ctypes.c_void_p)]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise ImportError(f"{_LIB_PATH} is not built: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(_LIB_PATH)
        P, U32, U64 = ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint64
        L.df11_encode.argtypes = [P, U64, ctypes.POINTER(EncodeOpts), ctypes.POINTER(HostTensorC)]
        L.df11_encode_group.argtypes = [ctypes.POINTER(P), ctypes.POINTER(U64), U32, ctypes.POINTER(EncodeOpts),
                                        ctypes.c_int, ctypes.POINTER(HostTensorC)]
        L.df11_host_tensor_free.argtypes = [ctypes.POINTER(HostTensorC)]
        L.df11_decompress.argtypes = [ctypes.POINTER(DeviceTensorC), P]
        L.df11_decompress_block.argtypes = [ctypes.POINTER(DeviceTensorC), U32, P]
        L.df11_decompress_block_ex.argtypes = [ctypes.POINTER(DeviceTensorC), U32, P, ctypes.c_int]
        L.df11_decompress_block_budget.argtypes = [ctypes.POINTER(DeviceTensorC), U32, P, ctypes.c_int, U32]
        L.df11_decompress_host.argtypes = [ctypes.POINTER(HostTensorC), ctypes.POINTER(DeviceTensorC), P, P]
        L.df11_plan_cta_ranges.argtypes = [P, U32, U32, U32, P]
        L.df11_plan_cta_ranges.restype = None
        L.df11_decompress_host_block.argtypes = [ctypes.POINTER(HostTensorC), ctypes.POINTER(DeviceTensorC),
                                                 ctypes.POINTER(P), U32, P, P]
        L.df11_histogram_device.argtypes = [P, U64, U32, P, P]
        L.df11_encode_plan_create.argtypes = [P, P, ctypes.POINTER(EncodeOpts), ctypes.POINTER(EncodePlanC)]
        L.df11_encode_plan_free.argtypes = [ctypes.POINTER(EncodePlanC)]
        L.df11_encode_device.argtypes = [P, ctypes.POINTER(EncodePlanC), ctypes.POINTER(DeviceBuffersC), P, U64, P]
        for f in ("df11_encode", "df11_encode_group", "df11_decompress", "df11_decompress_block",
                  "df11_decompress_block_ex", "df11_decompress_block_budget", "df11_decompress_host",
                  "df11_decompress_host_block",
                  "df11_histogram_device",
                  "df11_encode_plan_create", "df11_encode_device"):
            getattr(L, f).restype = ctypes.c_int
        L.df11_status_string.argtypes = [ctypes.c_int]
        L.df11_status_string.restype = ctypes.c_char_p
        L.df11_last_error_message.restype = ctypes.c_char_p
        L.df11_version.restype = ctypes.c_char_p
        L.df11_launch_count.argtypes = [ctypes.c_int]
        L.df11_launch_count.restype = ctypes.c_uint64
        L.df11_last_kernel_mask.argtypes = []
        L.df11_last_kernel_mask.restype = ctypes.c_uint32
        _lib = L
    return _lib


def _check(status: int):
    if status != DF11_OK:
        raise Df11Error(status, lib().df11_last_error_message().decode())


def library_path() -> str:
    return _LIB_PATH


def launch_count(reset: bool = False) -> int:
    return int(lib().df11_launch_count(1 if reset else 0))


def last_kernels() -> set:
    """Kernels this thread's last decompress call launched: a subset of {"alg1", "fast"}."""
    m = int(lib().df11_last_kernel_mask())
    return {k for b, k in ((1, "alg1"), (2, "fast")) if m & b}


# --------------------------------------------------------------------------- host side
class HostTensor:
    """A DF11 tensor in host memory (library-owned arrays exposed as numpy views)."""

    def __init__(self, c: HostTensorC, shape):
        self._c = c
        self.shape = tuple(shape)

    def __del__(self):
        try:
            lib().df11_host_tensor_free(ctypes.byref(self._c))
        except Exception:
            pass

    def _arr(self, name, count, dtype=np.uint8):
        p = getattr(self._c, name)
        if count == 0 or not p:
            return np.zeros(0, dtype)
        return np.ctypeslib.as_array(p, shape=(count,)).view(dtype) if dtype is np.uint8 else \
            np.ctypeslib.as_array(p, shape=(count,))

    num_elements = property(lambda s: int(s._c.num_elements))
    encoded_bits = property(lambda s: int(s._c.encoded_bits))
    T = property(lambda s: int(s._c.T))
    n = property(lambda s: int(s._c.n))
    B = property(lambda s: int(s._c.B))
    k = property(lambda s: int(s._c.k))
    lut_entry_bytes = property(lambda s: int(s._c.lut_entry_bytes))
    max_code_len = property(lambda s: int(s._c.max_code_len))
    value_format = property(lambda s: int(s._c.value_format))
    lut_bits = property(lambda s: int(s._c.lut_bits))

    @property
    def code_lengths(self):
        return np.frombuffer(bytes(self._c.code_lengths), np.uint8).copy()

    @property
    def luts(self):
        return self._arr("luts", int(self._c.luts_bytes))

    @property
    def encoded_exponent(self):
        return self._arr("encoded_exponent", int(self._c.encoded_exponent_bytes))

    @property
    def packed_sign_mantissa(self):
        return self._arr("packed_sign_mantissa", int(self._c.packed_sign_mantissa_bytes))

    @property
    def gaps(self):
        return self._arr("gaps", int(self._c.gaps_bytes))

    @property
    def block_output_pos(self):
        return self._arr("block_output_pos", self.B + 1, np.uint32)

    def compressed_bytes(self) -> int:
        """Bytes the method must read to rebuild the tensor (stream + sign/mantissa residuals + 5-bit
        gaps + BlockOutputPos + LUTs + CodeLengths), excluding alignment padding."""
        R = VALUE_FORMATS[VF_NAMES[self.value_format]][2]
        return ((self.encoded_bits + 7) // 8 + (R * self.num_elements + 7) // 8 + (5 * self.B * self.T + 7) // 8
                + 4 * (self.B + 1) + int(self._c.luts_bytes) + 256)

    def arrays(self) -> dict:
        return dict(code_lengths=self.code_lengths, luts=self.luts, encoded_exponent=self.encoded_exponent,
                    packed_sign_mantissa=self.packed_sign_mantissa, gaps=self.gaps,
                    block_output_pos=self.block_output_pos)


def _as_words(w, vf: str = "bf16") -> np.ndarray:
    """Host words of value format vf: uint16 (bf16/fp16) or uint8 (fp8) bit patterns."""
    wt = np.uint16 if VALUE_FORMATS[vf][1] == 2 else np.uint8
    try:
        import torch
        if isinstance(w, torch.Tensor):
            if w.is_cuda:
                raise ValueError("df11.encode takes a host tensor")
            w = w.contiguous()
            if w.element_size() != VALUE_FORMATS[vf][1]:
                raise ValueError(f"{vf} words are {VALUE_FORMATS[vf][1]} bytes")
            w = w.view(torch.int16 if wt is np.uint16 else torch.uint8)
            return w.numpy().view(wt)
    except ImportError:
        pass
    return np.ascontiguousarray(w).view(wt)


def _as_u16(w) -> np.ndarray:
    return _as_words(w, "bf16")


def _lut_bits(lut_bits) -> int:
    return LUT_BITS_MONOLITHIC if lut_bits == "mono" else int(lut_bits)


def _opts(T, n, lut_mode, num_threads, vf="bf16", lut_bits=8):
    return EncodeOpts(T, n, LUT_MODES[lut_mode], num_threads, VALUE_FORMATS[vf][0], _lut_bits(lut_bits))


def _infer_vf(w, vf):
    if vf is not None:
        return vf
    return {"torch.bfloat16": "bf16", "torch.float16": "fp16", "torch.float8_e4m3fn": "fp8_e4m3",
            "torch.float8_e5m2": "fp8_e5m2", "float16": "fp16"}.get(str(getattr(w, "dtype", "")), "bf16")


def encode(w, T: int = 256, n: int = 8, lut_mode: str = "auto", num_threads: int = 0, vf: str = None,
           lut_bits=8) -> HostTensor:
    """df11_encode: host tensor of value format vf -> HostTensor.  vf: "bf16" (torch.bfloat16 or uint16
    bit patterns; the default), "fp16", "fp8_e4m3" / "fp8_e5m2" (uint8 patterns); inferred from a torch
    (or numpy float16) dtype when not given.  lut_bits: b in [1, 16] or "mono"."""
    vf = _infer_vf(w, vf)
    a = _as_words(w, vf)
    shape = a.shape
    a = a.reshape(-1)
    c = HostTensorC()
    o = _opts(T, n, lut_mode, num_threads, vf, lut_bits)
    _check(lib().df11_encode(ctypes.c_void_p(a.ctypes.data if a.size else 0), a.size, ctypes.byref(o),
                             ctypes.byref(c)))
    return HostTensor(c, shape)


def encode_group(ws, T: int = 256, n: int = 8, lut_mode: str = "auto", shared_codebook: bool = False,
                 num_threads: int = 0, vf: str = None, lut_bits=8):
    vf = _infer_vf(ws[0], vf) if ws else "bf16"
    arrs = [_as_words(w, vf) for w in ws]
    shapes = [a.shape for a in arrs]
    flat = [a.reshape(-1) for a in arrs]
    cnt = len(flat)
    ptrs = (ctypes.c_void_p * cnt)(*[a.ctypes.data if a.size else None for a in flat])
    ns = (ctypes.c_uint64 * cnt)(*[a.size for a in flat])
    outs = (HostTensorC * cnt)()
    o = _opts(T, n, lut_mode, num_threads, vf, lut_bits)
    _check(lib().df11_encode_group(ptrs, ns, cnt, ctypes.byref(o), 1 if shared_codebook else 0, outs))
    res = []
    for i in range(cnt):
        c = HostTensorC()
        ctypes.memmove(ctypes.byref(c), ctypes.byref(outs[i]), ctypes.sizeof(HostTensorC))
        res.append(HostTensor(c, shapes[i]))
    return res


# --------------------------------------------------------------------------- device side
class DeviceTensor:
    """Device-resident DF11 tensor: torch uint8/int32 buffers + the C descriptor pointing at them."""

    def __init__(self, h: HostTensor, device="cuda", out=None):
        m = dict(num_elements=h.num_elements, T=h.T, n=h.n, B=h.B, k=h.k, lut_entry_bytes=h.lut_entry_bytes,
                 encoded_bits=h.encoded_bits, max_code_len=h.max_code_len, value_format=h.value_format,
                 lut_bits=h.lut_bits)
        self._init(m, h.arrays(), h.shape, device, out)

    @classmethod
    def from_arrays(cls, meta: dict, arrays: dict, shape=None, device="cuda", out=None) -> "DeviceTensor":
        """Upload DF11 arrays given as numpy (e.g. read from disk): keys code_lengths, luts,
        encoded_exponent, packed_sign_mantissa, gaps, block_output_pos; meta: num_elements, T, n, B, k,
        lut_entry_bytes, encoded_bits, max_code_len (+ value_format, lut_bits; default BF16, 8)."""
        self = cls.__new__(cls)
        self._init(meta, arrays, shape if shape is not None else (int(meta["num_elements"]),), device, out)
        return self

    def _init(self, meta, a, shape, device, out):
        import torch
        dev = torch.device(device)
        self.shape = tuple(shape)
        self.num_elements = int(meta["num_elements"])
        self.meta = {k: int(meta[k]) for k in ("T", "n", "B", "k", "lut_entry_bytes", "encoded_bits",
                                               "max_code_len")}
        self.meta["value_format"] = int(meta.get("value_format", 0))
        self.meta["lut_bits"] = int(meta.get("lut_bits", 8))
        self.vf = VF_NAMES[self.meta["value_format"]]
        B, T = self.meta["B"], self.meta["T"]
        R = VALUE_FORMATS[self.vf][2]
        self.compressed_bytes = ((self.meta["encoded_bits"] + 7) // 8 + (R * self.num_elements + 7) // 8
                                 + (5 * B * T + 7) // 8 + 4 * (B + 1) + int(np.asarray(a["luts"]).size) + 256)

        def up(x):
            t = torch.from_numpy(np.ascontiguousarray(x).view(np.uint8).copy())
            return t.to(dev, non_blocking=False)

        luts = np.asarray(a["luts"])
        self.encoded_exponent = up(a["encoded_exponent"])
        self.packed_sign_mantissa = up(a["packed_sign_mantissa"])
        self.gaps = up(a["gaps"])
        self.luts = up(luts if luts.size else np.zeros(16, np.uint8))
        self.code_lengths = up(a["code_lengths"])
        self.block_output_pos = up(np.asarray(a["block_output_pos"], np.uint32).view(np.uint8))
        self.out = out if out is not None else torch.empty(max(self.num_elements, 1), dtype=out_dtype(self.vf),
                                                           device=dev)

    def descriptor(self, out=None) -> DeviceTensorC:
        o = self.out if out is None else out
        if o.numel() < self.num_elements or o.element_size() != VALUE_FORMATS[self.vf][1]:
            raise ValueError(f"output buffer too small or not {VALUE_FORMATS[self.vf][1]}-byte words")
        m = self.meta
        return DeviceTensorC(self.encoded_exponent.data_ptr(), self.packed_sign_mantissa.data_ptr(),
                             self.gaps.data_ptr(), self.luts.data_ptr(), self.code_lengths.data_ptr(),
                             self.block_output_pos.data_ptr(), o.data_ptr(), self.num_elements,
                             m["T"], m["n"], m["B"], m["k"], m["lut_entry_bytes"], m["value_format"],
                             m["lut_bits"], 0)

    def staging_bytes(self) -> int:
        return sum(int(t.numel()) for t in (self.encoded_exponent, self.packed_sign_mantissa, self.gaps,
                                            self.luts, self.code_lengths, self.block_output_pos))


def clone_device_tensor(d: "DeviceTensor", out=None) -> "DeviceTensor":
    """A second device copy of a DF11 tensor (same format, fresh buffers; a new BF16 output unless
    `out` is given): e.g. to rotate over copies larger than L2 in timing loops."""
    c = DeviceTensor.__new__(DeviceTensor)
    c.__dict__.update(d.__dict__)
    for key in ("encoded_exponent", "packed_sign_mantissa", "gaps", "luts", "code_lengths", "block_output_pos"):
        setattr(c, key, getattr(d, key).clone())
    c.out = out if out is not None else d.out.clone()
    return c


def _u16_dtypes():
    import torch
    return (torch.bfloat16, torch.int16, torch.uint16)


def out_dtype(vf: str):
    """torch dtype of a decoded tensor of value format vf."""
    import torch
    return {"bf16": torch.bfloat16, "fp16": torch.float16, "fp8_e4m3": torch.float8_e4m3fn,
            "fp8_e5m2": torch.float8_e5m2}[vf]


def to_device(h: HostTensor, device="cuda", out=None) -> DeviceTensor:
    return DeviceTensor(h, device, out)


def _stream_ptr(stream):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return ctypes.c_void_p(s.cuda_stream)


def decompress(dt: DeviceTensor, out=None, stream=None, kernel: str = "auto"):
    """df11_decompress on the current (or given) stream; returns the BF16 tensor (shape restored)."""
    d = dt.descriptor(out)
    _check(lib().df11_decompress_block_ex(ctypes.byref(d), 1, _stream_ptr(stream), KERNELS[kernel]))
    o = dt.out if out is None else out
    return o[: dt.num_elements].view(dt.shape) if dt.num_elements else o[:0]


class BlockPlan:
    """Pre-marshalled descriptor array for repeated df11_decompress_block calls (no per-call Python
    work beyond one ctypes call)."""

    def __init__(self, dts, outs=None):
        if len(dts) > MAX_BATCH:
            raise ValueError("at most 64 tensors per block")
        self.dts = list(dts)
        self.outs = outs
        self.arr = (DeviceTensorC * max(len(dts), 1))()
        for i, dt in enumerate(self.dts):
            self.arr[i] = dt.descriptor(None if outs is None else outs[i])
        self.count = len(dts)

    def run(self, stream=None, kernel: str = "auto", max_ctas: int = 0):
        """One launch for the block (df11_decompress_block_budget; max_ctas = 0: every SM)."""
        _check(lib().df11_decompress_block_budget(self.arr, self.count, _stream_ptr(stream), KERNELS[kernel],
                                                  int(max_ctas)))

    def outputs(self):
        res = []
        for i, dt in enumerate(self.dts):
            o = dt.out if self.outs is None else self.outs[i]
            res.append(o[: dt.num_elements].view(dt.shape))
        return res


def decompress_block(dts, outs=None, stream=None, kernel: str = "auto", max_ctas: int = 0):
    """df11_decompress_block: every tensor of a transformer block in one launch; max_ctas
    caps the persistent grid (an SM budget for decode/compute overlap; 0 = every SM)."""
    plan = BlockPlan(dts, outs)
    plan.run(stream, kernel, max_ctas)
    return plan.outputs()


def decompress_host(h: HostTensor, dt: DeviceTensor, host_out, stream=None):
    """df11_decompress_host: H2D of h's arrays into dt's buffers, decode, D2H into host_out."""
    c_d = dt.descriptor()
    _check(lib().df11_decompress_host(ctypes.byref(h._c), ctypes.byref(c_d),
                                      ctypes.c_void_p(host_out.data_ptr()), _stream_ptr(stream)))
    return host_out


def decompress_host_block(hs, dts, host_outs, stream=None, copy_stream=None):
    """df11_decompress_host_block: the H2D + decode of tensor i+1 on `stream` overlap the D2H of tensor i
    on `copy_stream`; synchronising `stream` covers the whole block.  `hs` are HostTensor-like objects
    exposing a `_c` HostTensorC (pinned host arrays recommended)."""
    import torch
    n = len(hs)
    if copy_stream is None:
        copy_stream = torch.cuda.Stream()
    H = (HostTensorC * n)()
    D = (DeviceTensorC * n)()
    O = (ctypes.c_void_p * n)()
    for i, (h, dt, o) in enumerate(zip(hs, dts, host_outs)):
        ctypes.memmove(ctypes.byref(H, i * ctypes.sizeof(HostTensorC)), ctypes.byref(h._c), ctypes.sizeof(HostTensorC))
        D[i] = dt.descriptor()
        O[i] = o.data_ptr() if o is not None else None
    _check(lib().df11_decompress_host_block(H, D, O, n, _stream_ptr(stream), _stream_ptr(copy_stream)))
    return host_outs


# --------------------------------------------------------------------------- device encoder (NEXT-3)
class EncodePlan:
    """df11_encode_plan: codebook + geometry of one tensor (host); frees its LUT copy on deletion."""

    def __init__(self, codebook_hist, tensor_hist=None, T: int = 256, n: int = 8, lut_mode: str = "auto",
                 lut_bits=8, vf: str = "bf16"):
        cb = np.ascontiguousarray(codebook_hist, dtype=np.uint64)
        th = None if tensor_hist is None else np.ascontiguousarray(tensor_hist, dtype=np.uint64)
        if cb.shape != (256,) or (th is not None and th.shape != (256,)):
            raise ValueError("histograms have 256 bins")
        self._c = EncodePlanC()
        o = _opts(T, n, lut_mode, 0, vf, lut_bits)
        _check(lib().df11_encode_plan_create(ctypes.c_void_p(cb.ctypes.data),
                                             None if th is None else ctypes.c_void_p(th.ctypes.data),
                                             ctypes.byref(o), ctypes.byref(self._c)))

    def __del__(self):
        try:
            lib().df11_encode_plan_free(ctypes.byref(self._c))
        except Exception:
            pass

    def __getattr__(self, name):
        if name in ("num_elements", "encoded_bits", "T", "n", "B", "k", "lut_entry_bytes", "max_code_len", "lut_bits",
                    "value_format",
                    "luts_bytes", "encoded_exponent_bytes", "packed_sign_mantissa_bytes", "gaps_bytes",
                    "workspace_bytes"):
            return int(getattr(self.__dict__["_c"], name))
        raise AttributeError(name)

    @property
    def code_lengths(self):
        return np.frombuffer(bytes(self._c.code_lengths), np.uint8).copy()


_VF_OF_TORCH = {"torch.bfloat16": "bf16", "torch.float16": "fp16", "torch.float8_e4m3fn": "fp8_e4m3",
                "torch.float8_e5m2": "fp8_e5m2"}


def _dev_words(x, vf=None):
    """A contiguous CUDA tensor of words and its value format: BF16 / FP16 / FP8 dtypes name their
    format; int16 / uint16 / uint8 bit patterns need `vf` (default bf16 for 16-bit words)."""
    import torch
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise ValueError("expected a CUDA tensor")
    if vf is None:
        vf = _VF_OF_TORCH.get(str(x.dtype), "bf16" if x.element_size() == 2 else None)
        if vf is None:
            raise ValueError("pass vf= for 8-bit bit patterns")
    if x.element_size() != VALUE_FORMATS[vf][1]:
        raise ValueError(f"{vf} words are {VALUE_FORMATS[vf][1]} bytes")
    return x.contiguous(), vf


def _dev_u16(x):
    return _dev_words(x, "bf16")[0]


def _on(stream):
    """Context in which torch allocations, copies and read-backs run on `stream` (the current stream
    when None), so that buffers the library fills on that stream are ordered with everything around
    them (allocations are tied to the stream by the caching allocator)."""
    import contextlib
    import torch
    return torch.cuda.stream(stream) if stream is not None else contextlib.nullcontext()


def histogram_device(x, out=None, stream=None, vf=None):
    """df11_histogram_device: exponent histogram of a device tensor (BF16 / FP16 / FP8 words),
    accumulated into `out` (int64[256] on the same device; zeroed when created here).  Everything runs on
    `stream`."""
    import torch
    with _on(stream):
        x, vf = _dev_words(x, vf)
        if out is None:
            out = torch.zeros(256, dtype=torch.int64, device=x.device)
        _check(lib().df11_histogram_device(ctypes.c_void_p(x.data_ptr()), x.numel(), VALUE_FORMATS[vf][0],
                                           ctypes.c_void_p(out.data_ptr()), _stream_ptr(stream)))
    return out


def encode_device(x, T: int = 256, n: int = 8, lut_mode: str = "auto", codebook_hist=None, stream=None,
                  out=None, vf=None, lut_bits=8) -> "DeviceTensor":
    """GPU encoder: device tensor -> DeviceTensor (histogram on the GPU, codebook on the host, packing on
    the GPU).  Byte-identical to encode(x.cpu()) with the same options; with `codebook_hist` (host, 256
    bins, e.g. a group's summed histogram) the codebook is built from it."""
    with _on(stream):
        x, vf = _dev_words(x, vf)
        th = histogram_device(x, stream=stream, vf=vf).cpu().numpy().view(np.uint64)   # read back on `stream`
    plan = EncodePlan(th if codebook_hist is None else codebook_hist, th, T, n, lut_mode, lut_bits, vf)
    return encode_device_with_plan(x, plan, stream=stream, out=out)


def encode_device_with_plan(x, plan: EncodePlan, stream=None, out=None) -> "DeviceTensor":
    with _on(stream):
        return _encode_device_with_plan(x, plan, stream, out)


def _encode_device_with_plan(x, plan, stream, out):
    import torch
    vf = VF_NAMES[plan.value_format]
    x, _ = _dev_words(x, vf)
    if x.numel() != plan.num_elements:
        raise ValueError("tensor size does not match the plan")
    dev = x.device

    def buf(nbytes, zero=False):
        # small metadata buffers are zero-filled: the encoder writes their first nbytes only (the rest is
        # the 16-byte minimum allocation), and a host copy of the whole buffer must not read garbage
        n = max(int(nbytes), 16)
        return (torch.zeros if zero else torch.empty)(n, dtype=torch.uint8, device=dev)

    dt = DeviceTensor.__new__(DeviceTensor)
    dt.shape = tuple(x.shape)
    dt.num_elements = plan.num_elements
    dt.meta = {k: getattr(plan, k) for k in ("T", "n", "B", "k", "lut_entry_bytes", "encoded_bits", "max_code_len",
                                             "lut_bits")}
    dt.meta["value_format"] = plan.value_format
    dt.vf = vf
    dt.encoded_exponent = buf(plan.encoded_exponent_bytes)
    dt.packed_sign_mantissa = buf(plan.packed_sign_mantissa_bytes)
    dt.gaps = buf(plan.gaps_bytes)
    dt.luts = buf(plan.luts_bytes, zero=True)
    dt.code_lengths = buf(256)
    dt.block_output_pos = buf(4 * (plan.B + 1), zero=True)
    B, T = plan.B, plan.T
    R = VALUE_FORMATS[vf][2]
    dt.compressed_bytes = ((plan.encoded_bits + 7) // 8 + (R * plan.num_elements + 7) // 8 + (5 * B * T + 7) // 8
                           + 4 * (B + 1) + plan.luts_bytes + 256)
    dt.out = out if out is not None else torch.empty(max(plan.num_elements, 1), dtype=out_dtype(vf), device=dev)
    ws = buf(plan.workspace_bytes)
    d = DeviceBuffersC(dt.encoded_exponent.data_ptr(), dt.packed_sign_mantissa.data_ptr(), dt.gaps.data_ptr(),
                       dt.luts.data_ptr(), dt.code_lengths.data_ptr(), dt.block_output_pos.data_ptr())
    _check(lib().df11_encode_device(ctypes.c_void_p(x.data_ptr() if x.numel() else 0), ctypes.byref(plan._c),
                                    ctypes.byref(d), ctypes.c_void_p(ws.data_ptr()), ws.numel(),
                                    _stream_ptr(stream)))
    dt._workspace = ws     # keep alive until the stream has consumed it
    return dt


def encode_device_group(xs, T: int = 256, n: int = 8, lut_mode: str = "auto", shared_codebook: bool = True,
                        stream=None, vf=None, lut_bits=8):
    """GPU encoder for a group of tensors (e.g. one transformer block); shared_codebook builds one
    codebook from the summed histogram (R5)."""
    with _on(stream):
        hists = [histogram_device(x, stream=stream, vf=vf) for x in xs]
        hs = [h.cpu().numpy().view(np.uint64) for h in hists]
    total = np.sum(np.stack(hs), axis=0, dtype=np.uint64) if hs else np.zeros(256, np.uint64)
    res = []
    for x, h in zip(xs, hs):
        with _on(stream):
            x, xvf = _dev_words(x, vf)
        plan = EncodePlan(total if shared_codebook else h, h, T, n, lut_mode, lut_bits, xvf)
        res.append(encode_device_with_plan(x, plan, stream=stream))
    return res
