"""ctypes binding of libssn_b200.so (the C ABI declared in include/ssn.h).

The product path has NO CPU fallback: if the CUDA library is missing or no CUDA device
is present, every compute call raises SsnUnavailable.  `build()` compiles the library
in-tree with nvcc for sm_100a.
"""

import ctypes
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB_PATH = os.path.join(HERE, "libssn_b200.so")
if os.environ.get("SSN_LIB"):             # experiments only: an alternative build of the same sources
    LIB_PATH = os.environ["SSN_LIB"]
CSRC = os.path.join(HERE, "csrc")
SOURCES = ["ssn_elementwise.cu", "ssn_gemm_simt.cu", "ssn_gemm_tc.cu", "ssn_chain.cu"]
NVCC_FLAGS = ["-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-lineinfo", "-std=c++17",
              "-Xcompiler", "-fPIC", "-shared"]

SSN_ERR_ARG, SSN_ERR_CUDA, SSN_ERR_UNSUPPORTED = -1, -2, -3


class SsnUnavailable(RuntimeError):
    """The CUDA extension (or a CUDA device) is missing; there is no CPU fallback."""


class SsnKernelError(RuntimeError):
    pass


def build(force=False, verbose=False):
    srcs = [os.path.join(CSRC, s) for s in SOURCES if os.path.exists(os.path.join(CSRC, s))]
    deps = srcs + [os.path.join(CSRC, f) for f in os.listdir(CSRC) if f.endswith((".cuh", ".h"))]
    deps.append(os.path.join(ROOT, "include", "ssn.h"))
    if (not force and os.path.exists(LIB_PATH)
            and os.path.getmtime(LIB_PATH) >= max(os.path.getmtime(d) for d in deps)):
        return LIB_PATH
    cmd = ["nvcc", *NVCC_FLAGS, "-I" + os.path.join(ROOT, "include"), "-I" + CSRC, *srcs,
           "-lcuda", "-o", LIB_PATH]
    if verbose:
        print(" ".join(cmd))
    subprocess.check_call(cmd)
    return LIB_PATH


_U64, _I64, _I32, _P = ctypes.c_uint64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p

_SIGS = {
    "ssn_version": [],
    "ssn_kernel_launches": [],
    "ssn_ewise": [_I32, _P, _P, _P, _U64, _U64, _U64, _U64, _U64, _U64, _P],
    "ssn_gen": [_P, _U64, _P, _U64, _U64, _U64, _I32, _P, _I32, _P, _U64, _U64, _U64, _I32, _U64, _P],
    "ssn_rec": [_P, _U64, _U64, _P, _I32, _P, _U64, _U64, _I32, _U64, _P],
    "ssn_reduce_apply": [_P, _U64, _U64, _I32, _P, _I32, _P, _U64, _U64, _U64, _I32, _U64, _P],
    "ssn_reshare_finish": [_P, _U64, _U64, _P, _I32, _P, _U64, _P, _U64, _U64, _U64, _P, _U64, _P, _U64,
                           _U64, _I32, _U64, _P],
    "ssn_trunc_elite": [_P, _U64, _I32, _I32, _P, _P, _I64, _I64, _I64, _P, _U64, _U64, _I32, _P, _I32, _P,
                        _U64, _P, _U64, _U64, _P],
    "ssn_nonlin_elite": [_P, _U64, _I32, _P, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _U64, _P],
    "ssn_encode_signed": [_P, _P, _U64, _P, _U64, _P],
    "ssn_decode_signed": [_P, _P, _U64, _U64, _P],
    "ssn_inv": [_P, _P, _U64, _U64, _P],
    "ssn_rand": [_P, _U64, _U64, _U64, _U64, _U64, _P],
    "ssn_mask_trunc": [_U64, _U64, _U64, _U64, _U64, _I32, _P, _I32, _P, _P, _U64, _U64, _P],
    "ssn_mask_beta": [_I32, _I32, _I32, _I32, _I32, _I32, _U64, _U64, _U64, _I32, _P, _I32, _P, _U64, _P,
                      _U64, _U64, _P],
    "ssn_window_gather": [_P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P],
    "ssn_pool_expand": [_P, _P, _I32, _I32, _I32, _I32, _I32, _I32, _P],
    "ssn_conv_simt": [_P, _U64, _P, _U64, _P, _U64, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32,
                      _I32, _U64, _P],
    "ssn_dense_simt": [_P, _U64, _P, _U64, _P, _U64, _I32, _I32, _I32, _I32, _U64, _P],
    "ssn_limb_split": [_P, _U64, _U64, _U64, _I32, _P, _U64, _I32, _P],
    "ssn_im2col_limbs": [_P, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _U64, _U64, _P],
    "ssn_gemm_tc": [_P, _P, _I32, _I32, _I32, _I32, _U64, _U64, _P, _U64, _U64, _P],
    "ssn_layer_chain": [_P, _P],
    "ssn_gemm_tc_conv": [_P, _I32, _I32, _I32, _I32, _I32, _I32, _P, _I32, _I32, _P, _U64, _U64, _P],
    "ssn_planes_shift": [_P, _U64, _I32, _P],
    "ssn_mma_peak": [_I32, _I32, _P, _P, _P],
    "ssn_mma_probe": [_I32, _I32, _I32, _I32, _P, _P, _P],
    "ssn_gemm_tc_subshares": [_P, _P, _I32, _I32, _I32, _U64, _U64, _P, _U64, _P],
    "ssn_planes_cn": [_P, _I32, _I32, _I32, _I32, _I32, _I32, _I32, _P, _U64, _I32, _P],
    "ssn_chain_supported": [_I32, _I32, _P, _U64],
    "ssn_inv_table": [_P, _U64, _U64, _P],
}


class ChainDesc(ctypes.Structure):
    """struct ssn_chain_desc (include/ssn.h)."""
    _fields_ = [
        ("acc", _P), ("acc_pstride", _U64),
        ("bias", _P), ("bias_pstride", _U64), ("bias_div", _U64), ("bias_mod", _U64),
        ("other", _P), ("other_pstride", _U64),
        ("out", _P), ("out_pstride", _U64),
        ("nel", _U64),
        ("nout", _I32),
        ("value_bound", _I64), ("r", _I64), ("d", _I64),
        ("emax", _U64),
        ("verify", _I32),
        ("fail", _P),
        ("nonlin", _I32), ("relu", _I32), ("pool_kind", _I32), ("nb", _I32), ("c", _I32), ("h", _I32),
        ("w", _I32), ("kh", _I32), ("kw", _I32), ("fan", _I32),
        ("bmax", _U64),
        ("party_seed", _U64), ("party_stream", _U64), ("src_seed", _U64), ("src_stream", _U64),
        ("k", _I32), ("n", _I32),
        ("ids", _P), ("rt", _P), ("ext", _P),
        ("p", _U64),
        ("fault_rank", _I32),
        ("planes", _P),
        ("plane_pstride", _U64), ("plane_lstride", _U64), ("plane_cstride", _U64), ("plane_istride", _U64),
        ("plane_wp", _I32), ("plane_copies", _I32), ("plane_nparty", _I32),
        ("scratch", _P),
        ("inv_table", _P), ("inv_table_len", _U64),
        ("nonlin_only", _I32),
        ("host_masks", _I32),
        ("h_zero", _P), ("h_alpha", _P), ("h_comp", _P), ("h_tcoef", _P), ("h_beta", _P), ("h_binv", _P),
        ("h_period", _U64), ("h_period_out", _U64),
        ("h_period_in", _U64),
        ("gather", _I32), ("gather_h", _I32), ("gather_w", _I32), ("gather_stride", _I32), ("gather_pad", _I32),
    ]

_lib = None


def exported_symbols():
    return list(_SIGS)


def load(require_cuda=True):
    """Load the library (no device needed).  Raises SsnUnavailable if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise SsnUnavailable(f"{LIB_PATH} is missing: run __graft_entry__.build() "
                                 "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        for name, args in _SIGS.items():
            fn = getattr(L, name, None)
            if fn is None and os.environ.get("SSN_LIB"):     # an older experimental build
                continue
            if fn is None:
                raise SsnUnavailable(f"{LIB_PATH} does not export {name}: rebuild it")
            fn.argtypes = args
            fn.restype = ctypes.c_uint64 if name == "ssn_kernel_launches" else ctypes.c_int
        _lib = L
    if require_cuda and not torch.cuda.is_available():
        raise SsnUnavailable("no CUDA device: the SSNet B200 path has no CPU fallback")
    return _lib


def launch_count():
    """Kernels launched by libssn_b200 in this process (the library's own counter, incremented
    at every launch site; an entry point may launch more than one kernel)."""
    return int(load(require_cuda=False).ssn_kernel_launches())


def call(name, *args):
    rc = getattr(load(), name)(*args)
    if rc != 0:
        if rc == SSN_ERR_ARG:
            raise ValueError(f"{name}: invalid arguments")
        raise SsnKernelError(f"{name} failed with code {rc}")


class SubshareDesc(ctypes.Structure):
    """ssn_subshare_desc (include/ssn.h)."""
    _fields_ = [("sub", ctypes.c_uint64), ("party_stride", ctypes.c_uint64), ("front_stride", ctypes.c_uint64),
                ("seed", ctypes.c_uint64), ("stream", ctypes.c_uint64), ("km1", ctypes.c_int), ("nf", ctypes.c_int),
                ("front_ids", ctypes.c_uint64)]


def stream_ptr():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def ptr(t):
    """Device pointer of a tensor (None -> NULL)."""
    if t is None:
        return None
    return ctypes.c_void_p(t.data_ptr())


def u64_array(vals):
    arr = (ctypes.c_uint64 * max(1, len(vals)))(*[int(v) for v in vals])
    return arr
