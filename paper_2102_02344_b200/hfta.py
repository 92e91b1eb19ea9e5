"""Thin ctypes binding of libhfta (include/hfta.h) -- argument marshalling only.

Every function here has the name of its C entry point and forwards plain
integers / device pointers; all arithmetic of the hot path runs in the
library's sm_100a kernels.  There is no fallback: if libhfta.so is missing
or cannot be loaded, importing this module raises.

Tensor helpers `tin(t, bstride, ld)` / `tout(...)` build the hfta_in /
hfta_out structs from torch tensors (PyTorch is plumbing: memory + streams).
"""
import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libhfta.so")

if not os.path.exists(LIB_PATH):
    raise ImportError("libhfta.so not built at %s: run `python -m paper_2102_02344_b200.build` "
                      "(no CPU fallback exists)" % LIB_PATH)
_lib = C.CDLL(LIB_PATH)

HFTA_F32, HFTA_BF16, HFTA_BF16_F32 = 0, 1, 2
ACT_NONE, ACT_RELU, ACT_LEAKY_RELU, ACT_TANH, ACT_SIGMOID = 0, 1, 2, 3, 4
STATUS = {0: "HFTA_OK", 1: "HFTA_ERR_INVALID_VALUE", 2: "HFTA_ERR_SHAPE", 3: "HFTA_ERR_ALIGNMENT",
          4: "HFTA_ERR_UNSUPPORTED", 5: "HFTA_ERR_ARCH", 6: "HFTA_ERR_WORKSPACE", 7: "HFTA_ERR_CUDA",
          8: "HFTA_ERR_NOT_INITIALIZED"}
(HFTA_ERR_INVALID_VALUE, HFTA_ERR_SHAPE, HFTA_ERR_ALIGNMENT, HFTA_ERR_UNSUPPORTED, HFTA_ERR_ARCH, HFTA_ERR_WORKSPACE,
 HFTA_ERR_CUDA, HFTA_ERR_NOT_INITIALIZED) = range(1, 9)


class HftaError(RuntimeError):
    def __init__(self, code, fn, msg):
        super().__init__("%s -> %s: %s" % (fn, STATUS.get(code, code), msg))
        self.code = code


class hfta_in(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("bstride", C.c_int64), ("ld", C.c_int64)]


class hfta_out(C.Structure):
    _fields_ = [("ptr", C.c_void_p), ("bstride", C.c_int64), ("ld", C.c_int64)]


class hfta_conv_desc(C.Structure):
    _fields_ = [(n, C.c_int) for n in ("N", "H", "W", "C_in", "C_out", "kh", "kw", "stride", "pad", "transposed")]


i32, i64, u64, f32, vp, sz = C.c_int, C.c_int64, C.c_uint64, C.c_float, C.c_void_p, C.c_size_t

# name -> (restype, argtypes); the exported symbol list of include/hfta.h
_SIGS = {
    "hfta_init": (i32, [i32]),
    "hfta_last_error": (C.c_char_p, []),
    "hfta_version": (C.c_char_p, []),
    "hfta_launch_count": (u64, []),
    "hfta_fused_linear_fwd": (i32, [i32, i64, i64, i64, i32, hfta_in, hfta_in, vp, i64, i64, i64, hfta_out, vp]),
    "hfta_fused_linear_bwd_workspace": (sz, [i32, i64, i64, i64, i32]),
    "hfta_fused_linear_bwd": (i32, [i32, i64, i64, i64, i32, hfta_in, hfta_in, hfta_in, hfta_out, vp, i64, i64, vp,
                                    i64, i32, vp, sz, vp]),
    "hfta_linear_colstat_size": (sz, [i32, i64, i64]),
    "hfta_fused_linear_fwd_stats": (i32, [i32, i64, i64, i64, hfta_in, hfta_in, vp, i64, i64, i64, hfta_out, vp, vp]),
    "hfta_fused_bn_fwd_colstat": (i32, [i32, i64, i64, i32, hfta_in, vp, vp, i64, vp, vp, f32, f32, i32, f32, hfta_out,
                                        vp, vp, vp, vp]),
    "hfta_fused_bn_workspace": (sz, [i32, i64, i64]),
    "hfta_fused_bn_fwd": (i32, [i32, i64, i64, i32, hfta_in, vp, vp, i64, vp, vp, f32, f32, i32, f32, hfta_out, vp,
                                vp, vp, sz, vp]),
    "hfta_fused_bn_bwd": (i32, [i32, i64, i64, i32, hfta_in, hfta_in, vp, vp, i64, vp, vp, i32, f32, hfta_out, vp, vp,
                                i32, vp, sz, vp]),
    "hfta_bn_max_fwd": (i32, [i32, i64, i64, i64, i32, hfta_in, vp, vp, i64, vp, vp, i32, f32, hfta_out, vp, vp]),
    "hfta_bn_max_bwd_workspace": (sz, [i32, i64, i64]),
    "hfta_bn_max_bwd": (i32, [i32, i64, i64, i64, i32, hfta_in, hfta_in, vp, vp, vp, i64, vp, vp, i32, f32, hfta_out,
                              vp, vp, vp, sz, vp]),
    "hfta_fused_linear_bn_max_workspace": (sz, [i32, i64, i64, i64, i64]),
    "hfta_fused_linear_bn_max_fwd": (i32, [i32, i64, i64, i64, i64, i32, hfta_in, hfta_in, vp, i64, vp, vp, i64, vp,
                                           vp, f32, f32, i32, f32, hfta_out, vp, hfta_out, vp, vp, vp, vp, vp, sz,
                                           vp]),
    "hfta_fused_linear_bn_max_bwd": (i32, [i32, i64, i64, i64, i64, i32, hfta_in, hfta_in, hfta_in, vp, hfta_in, vp,
                                           i64, vp, vp, i64, vp, vp, vp, vp, i32, f32, hfta_out, i32, f32, vp, i64,
                                           i64, vp, i64, vp, vp, i32, vp, sz, vp]),
    "hfta_fused_linear_bn_workspace": (sz, [i32, i64, i64, i64]),
    "hfta_fused_linear_bn_fwd": (i32, [i32, i64, i64, i64, i32, hfta_in, hfta_in, vp, i64, vp, vp, i64, vp, vp, f32,
                                       f32, i32, f32, hfta_out, vp, vp, vp, vp, vp, sz, vp]),
    "hfta_fused_linear_bn_bwd": (i32, [i32, i64, i64, i64, i32, hfta_in, hfta_in, hfta_in, vp, i64, vp, i64, vp, vp,
                                       vp, vp, hfta_out, i32, f32, vp, i64, i64, vp, i64, vp, vp, i32, vp, sz, vp]),
    "hfta_transform_points_fwd": (i32, [i32, i64, i64, i32, hfta_in, hfta_in, i32, hfta_out, vp]),
    "hfta_transform_points_bwd": (i32, [i32, i64, i64, i32, hfta_in, hfta_in, hfta_out, vp]),
    "hfta_dropout_fwd": (i32, [i32, i64, i64, i32, hfta_in, hfta_out, u64, i64, vp, C.c_int32, f32, C.c_int32, vp,
                               vp]),
    "hfta_dropout_bwd": (i32, [i32, i64, i64, i32, hfta_in, hfta_out, u64, i64, vp, C.c_int32, f32, C.c_int32, vp,
                               vp]),
    "hfta_colsum_workspace": (sz, [i32, i64, i64, i64]),
    "hfta_colsum": (i32, [i32, i64, i64, i64, i32, hfta_in, vp, i64, i32, vp, sz, vp]),
    "hfta_loss_workspace": (sz, [i32, i64]),
    "hfta_loss_nll": (i32, [i32, i64, i64, i32, hfta_in, vp, i64, vp, vp, hfta_out, vp, sz, vp]),
    "hfta_loss_mse": (i32, [i32, i64, i64, i32, hfta_in, vp, i64, i64, vp, vp, hfta_out, vp, sz, vp]),
    "hfta_fused_adam": (i32, [i32, i64, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, vp, vp, i64, vp]),
    "hfta_cast_f32_bf16": (i32, [i64, vp, vp, vp]),
    "hfta_step_increment": (i32, [vp, vp]),
    "hfta_add": (i32, [i32, i64, i64, i32, hfta_in, hfta_in, hfta_out, vp]),
    "hfta_feature_transform_make": (i32, [i32, i64, i64, i32, vp, i64, hfta_out, vp]),
    "hfta_feature_transform_reg_workspace": (sz, [i32, i64]),
    "hfta_feature_transform_reg": (i32, [i32, i64, i64, vp, i64, vp, i64, f32, vp, i64, vp, vp, vp, sz, vp]),
    "hfta_fused_conv_workspace": (sz, [i32, C.POINTER(hfta_conv_desc), i32]),
    "hfta_fused_conv_fwd": (i32, [i32, C.POINTER(hfta_conv_desc), i32, hfta_in, hfta_in, hfta_out, i32, f32, vp, sz,
                                  vp]),
    "hfta_fused_conv_bwd": (i32, [i32, C.POINTER(hfta_conv_desc), i32, hfta_in, hfta_in, hfta_in, hfta_out, vp, i64,
                                  i32, vp, sz, vp]),
    "hfta_fused_conv_fwd_stats": (i32, [i32, C.POINTER(hfta_conv_desc), i32, hfta_in, hfta_in, hfta_out, vp, vp, sz,
                                        vp]),
    "hfta_fused_conv_bwd_gated": (i32, [i32, C.POINTER(hfta_conv_desc), i32, hfta_in, hfta_in, hfta_in, hfta_out, vp,
                                        i64, i32, i32, f32, hfta_in, vp, sz, vp]),
    "hfta_loss_bce_logits": (i32, [i32, i64, i32, hfta_in, f32, vp, vp, hfta_out, vp, sz, vp]),
    "hfta_act_fwd": (i32, [i32, i64, i64, i32, i32, f32, hfta_in, hfta_out, vp]),
    "hfta_act_bwd": (i32, [i32, i64, i64, i32, i32, f32, hfta_in, hfta_in, hfta_out, vp]),
    "hfta_fused_sgd": (i32, [i32, i64, vp, vp, vp, i64, vp, vp, vp, vp, i32, vp, vp, i64, vp]),
    "hfta_fused_adadelta": (i32, [i32, i64, vp, vp, vp, vp, i64, vp, vp, vp, vp, vp, i64, vp]),
    "hfta_steplr": (i32, [i32, vp, vp, vp, i64, vp, vp]),
    "hfta_maxpool2d_fwd": (i32, [i32, i32, i32, i32, i32, i32, i32, i32, i32, hfta_in, hfta_out, vp, i64, vp]),
    "hfta_maxpool2d_bwd": (i32, [i32, i32, i32, i32, i32, i32, i32, i32, i32, hfta_in, vp, i64, hfta_out, vp]),
    "hfta_avgpool2d_fwd": (i32, [i32, i64, i64, i64, i32, hfta_in, hfta_out, vp]),
    "hfta_avgpool2d_bwd": (i32, [i32, i64, i64, i64, i32, hfta_in, hfta_out, vp]),
}

EXPORTED = sorted(_SIGS)


def _wrap(name, restype, argtypes):
    fn = getattr(_lib, name)
    fn.restype = restype
    fn.argtypes = argtypes
    if restype is not i32:
        return fn

    def call(*args):
        st = fn(*args)
        if st != 0:
            raise HftaError(st, name, _lib.hfta_last_error().decode())
        return st
    call.__name__ = name
    return call


for _n, (_r, _a) in _SIGS.items():
    globals()[_n] = _wrap(_n, _r, _a)
_lib.hfta_last_error.restype = C.c_char_p


# ------------------------------------------------------------- helpers ----

def ptr(t):
    """Device pointer of a torch tensor (or None/int passthrough)."""
    if t is None:
        return None
    if isinstance(t, int):
        return t
    return t.data_ptr()


def tin(t, bstride, ld, offset=0):
    """hfta_in over tensor t, element offset `offset` (in t's dtype)."""
    return hfta_in(ptr(t) + offset * t.element_size(), int(bstride), int(ld))


def tout(t, bstride, ld, offset=0):
    if t is None:
        return hfta_out(None, 0, 1)
    return hfta_out(ptr(t) + offset * t.element_size(), int(bstride), int(ld))


def stream_ptr(stream=None):
    import torch
    s = torch.cuda.current_stream() if stream is None else stream
    return s.cuda_stream


def version():
    return _lib.hfta_version().decode()
