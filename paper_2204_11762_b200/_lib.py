"""Thin Python binding of libmfa.so (include/mfa.h): argument marshalling only.

Every step of the hot path runs in the library's sm_100a kernels; PyTorch is
used for device memory and streams.  There is no fallback: if libmfa.so is
missing or no CUDA device is present, the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libmfa.so")

MFA_OK = 0
STATUS = {0: "MFA_OK", 1: "MFA_ERR_INVALID_ARG", 2: "MFA_ERR_KNOTS", 3: "MFA_ERR_UNSUPPORTED",
          4: "MFA_ERR_DOMAIN", 5: "MFA_ERR_CUDA", 6: "MFA_ERR_OOM", 7: "MFA_ERR_DEVICE"}
TILE = 16
LAYOUTS = {"auto": 0, "quads": 1, "bezier": 2, "bricks": 3, "bezier_grouped": 4}

# C-ABI symbols declared in include/mfa.h (checked by tests/test_abi.py)
EXPORTS = ("mfa_model_create", "mfa_model_create_ex", "mfa_model_info", "mfa_model_destroy", "mfa_eval_batch", "mfa_render",
           "mfa_render_host", "mfa_render_host_views", "mfa_unpack_tiles", "mfa_last_error", "mfa_version",
           "mfa_render_field", "mfa_image_quality", "mfa_image_quality_workspace", "mfa_eval_hessian",
           "mfa_fit_grid", "mfa_encode_grid", "mfa_eval_batch_ws", "mfa_eval_workspace_bytes", "mfa_render_ex",
           "mfa_eval_hessian_ws", "mfa_hessian_workspace_bytes", "mfa_enable_peer_access",
           "mfa_ipc_open", "mfa_ipc_close", "mfa_ipc_alloc", "mfa_ipc_free", "mfa_probe_fp32", "mfa_probe_read_bw")


class MfaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


class Camera_t(C.Structure):
    _fields_ = [("eye", C.c_double * 3), ("look_at", C.c_double * 3), ("up", C.c_double * 3),
                ("fov_y_deg", C.c_double), ("ortho_half_height", C.c_double),
                ("width", C.c_int32), ("height", C.c_int32)]


class TF_t(C.Structure):
    _fields_ = [("rgba", C.c_void_p), ("n_entries", C.c_int32), ("v_lo", C.c_float), ("v_hi", C.c_float)]


class RenderParams_t(C.Structure):
    _fields_ = [("box_min", C.c_double * 3), ("box_max", C.c_double * 3), ("step", C.c_double),
                ("o_max", C.c_double), ("shading", C.c_int32), ("ka", C.c_double), ("kd", C.c_double),
                ("ks", C.c_double), ("shininess", C.c_double), ("grad_eps", C.c_double),
                ("out_fp16", C.c_int32)]


class Tiles_t(C.Structure):
    _fields_ = [("n_tiles", C.c_int64), ("tiles", C.c_void_p), ("scatter", C.c_int32)]


class ModelDesc_t(C.Structure):
    _fields_ = [("degree", C.c_int32 * 3), ("nctrl", C.c_int64 * 3), ("uniform", C.c_int32 * 3),
                ("v_min", C.c_float), ("v_max", C.c_float), ("device_bytes", C.c_int64),
                ("device", C.c_int32), ("layout", C.c_int32), ("model_bytes", C.c_int64),
                ("create_ms", C.c_double)]


class Field_t(C.Structure):
    _fields_ = [("kind", C.c_int32), ("value_src", C.c_int32), ("grad_src", C.c_int32),
                ("prm", C.c_double * 6)]


class RenderExt_t(C.Structure):
    _fields_ = [("field", C.POINTER(Field_t)), ("n_lights", C.c_int32), ("light_dir", C.POINTER(C.c_double)),
                ("light_intensity", C.POINTER(C.c_double)), ("curv_rgba", C.c_void_p), ("curv_n", C.c_int32),
                ("curv_range", C.c_double)]


class EncodeConfig_t(C.Structure):
    _fields_ = [("degree", C.c_int32), ("nctrl_init", C.c_int64 * 3), ("e_max", C.c_double),
                ("max_rounds", C.c_int32), ("max_ctrl", C.c_int64 * 3)]


class EncodeResult_t(C.Structure):
    _fields_ = [("nctrl", C.c_int64 * 3), ("rounds", C.c_int32), ("converged", C.c_int32),
                ("max_err", C.c_double), ("rms_err", C.c_double)]


class ModelOptions_t(C.Structure):
    _fields_ = [("layout", C.c_int32)]


_lib = None


def lib():
    """Load libmfa.so (raises if it is missing -- no CPU fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} not built: run `python -m paper_2204_11762_b200.build` "
                              "(there is no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        vp, i32, i64 = C.c_void_p, C.c_int32, C.c_int64
        L.mfa_model_create.restype = C.c_int
        L.mfa_model_create.argtypes = [C.POINTER(i32), C.POINTER(i64), C.POINTER(C.POINTER(C.c_double)), vp, i32,
                                       vp, C.POINTER(vp)]
        L.mfa_model_create_ex.restype = C.c_int
        L.mfa_model_create_ex.argtypes = [C.POINTER(i32), C.POINTER(i64), C.POINTER(C.POINTER(C.c_double)), vp,
                                          i32, C.POINTER(ModelOptions_t), vp, C.POINTER(vp)]
        L.mfa_model_info.restype = C.c_int
        L.mfa_model_info.argtypes = [vp, C.POINTER(ModelDesc_t)]
        L.mfa_model_destroy.restype = C.c_int
        L.mfa_model_destroy.argtypes = [vp]
        L.mfa_eval_batch.restype = C.c_int
        L.mfa_eval_batch.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.mfa_eval_workspace_bytes.restype = C.c_size_t
        L.mfa_eval_workspace_bytes.argtypes = [vp, i64]
        L.mfa_eval_batch_ws.restype = C.c_int
        L.mfa_eval_batch_ws.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp]
        L.mfa_hessian_workspace_bytes.restype = C.c_size_t
        L.mfa_hessian_workspace_bytes.argtypes = [vp, i64]
        L.mfa_eval_hessian_ws.restype = C.c_int
        L.mfa_eval_hessian_ws.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp, C.c_size_t, vp]
        L.mfa_eval_hessian.restype = C.c_int
        L.mfa_eval_hessian.argtypes = [vp, i64, vp, vp, vp, vp, vp, vp, vp, vp]
        L.mfa_render.restype = C.c_int
        L.mfa_render.argtypes = [vp, i32, C.POINTER(Camera_t), C.POINTER(TF_t), C.POINTER(RenderParams_t),
                                 C.POINTER(Tiles_t), vp, vp, vp]
        L.mfa_fit_grid.restype = C.c_int
        L.mfa_fit_grid.argtypes = [C.POINTER(i64), vp, i32, C.POINTER(i64), C.POINTER(C.POINTER(C.c_double)), vp,
                                   vp, vp]
        L.mfa_encode_grid.restype = C.c_int
        L.mfa_encode_grid.argtypes = [C.POINTER(i64), vp, C.POINTER(EncodeConfig_t),
                                      C.POINTER(C.POINTER(C.c_double)), vp, C.POINTER(EncodeResult_t), vp, vp]
        L.mfa_enable_peer_access.restype = C.c_int
        L.mfa_enable_peer_access.argtypes = [i32]
        L.mfa_ipc_open.restype = C.c_int
        L.mfa_ipc_open.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.mfa_ipc_close.restype = C.c_int
        L.mfa_ipc_close.argtypes = [C.c_void_p]
        L.mfa_render_ex.restype = C.c_int
        L.mfa_render_ex.argtypes = [vp, i32, C.POINTER(Camera_t), C.POINTER(TF_t), C.POINTER(RenderParams_t),
                                    C.POINTER(RenderExt_t), C.POINTER(Tiles_t), vp, vp, vp]
        L.mfa_render_field.restype = C.c_int
        L.mfa_render_field.argtypes = [vp, i32, C.POINTER(Camera_t), C.POINTER(TF_t), C.POINTER(RenderParams_t),
                                       C.POINTER(Field_t), C.POINTER(Tiles_t), vp, vp, vp]
        L.mfa_image_quality_workspace.restype = C.c_size_t
        L.mfa_image_quality_workspace.argtypes = [i32, i32]
        L.mfa_image_quality.restype = C.c_int
        L.mfa_image_quality.argtypes = [i32, i32, vp, vp, vp, vp, C.c_size_t, vp, vp]
        L.mfa_render_host.restype = C.c_int
        L.mfa_render_host.argtypes = [vp, i32, C.POINTER(Camera_t), vp, i32, C.c_float, C.c_float,
                                      C.POINTER(RenderParams_t), vp, vp, vp]
        L.mfa_render_host_views.restype = C.c_int
        L.mfa_render_host_views.argtypes = [vp, i32, C.POINTER(Camera_t), vp, i32, C.c_float, C.c_float,
                                            C.POINTER(RenderParams_t), C.POINTER(C.c_void_p), vp, vp]
        L.mfa_ipc_alloc.restype = C.c_int
        L.mfa_ipc_alloc.argtypes = [C.c_size_t, C.POINTER(C.c_void_p), C.c_char_p]
        L.mfa_ipc_free.restype = C.c_int
        L.mfa_ipc_free.argtypes = [vp]
        L.mfa_unpack_tiles.restype = C.c_int
        L.mfa_unpack_tiles.argtypes = [vp, i32, vp, i64, i32, i32, i32, vp, vp]
        L.mfa_last_error.restype = C.c_char_p
        L.mfa_last_error.argtypes = []
        L.mfa_version.restype = C.c_char_p
        L.mfa_version.argtypes = []
        L.mfa_probe_fp32.restype = C.c_int
        L.mfa_probe_fp32.argtypes = [i32, C.POINTER(C.c_double)]
        L.mfa_probe_read_bw.restype = C.c_int
        L.mfa_probe_read_bw.argtypes = [i64, i32, C.POINTER(C.c_double)]
        _lib = L
    return _lib


def _check(st: int):
    if st != MFA_OK:
        raise MfaError(st, lib().mfa_last_error().decode())


def _stream_ptr(stream=None):
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def _ptr(t):
    return C.c_void_p(t.data_ptr()) if t is not None else C.c_void_p(0)


def cameras_t(cams):
    arr = (Camera_t * len(cams))()
    for i, c in enumerate(cams):
        for k in range(3):
            arr[i].eye[k] = c.eye[k]
            arr[i].look_at[k] = c.look_at[k]
            arr[i].up[k] = c.up[k]
        arr[i].fov_y_deg = c.fov_y_deg
        arr[i].ortho_half_height = c.ortho_half_height
        arr[i].width = c.width
        arr[i].height = c.height
    return arr


def field_t(f):
    """f: workloads.AnalyticField (kind, value_src, grad_src, prm) -> mfa_field."""
    r = Field_t()
    r.kind, r.value_src, r.grad_src = int(f.kind), int(f.value_src), int(f.grad_src)
    for i, x in enumerate(f.prm):
        r.prm[i] = float(x)
    return r


def params_t(p, out_fp16=False):
    r = RenderParams_t()
    for k in range(3):
        r.box_min[k] = p.box_min[k]
        r.box_max[k] = p.box_max[k]
    r.step = p.step
    r.o_max = p.o_max
    r.shading = int(p.shading)
    r.ka, r.kd, r.ks, r.shininess = p.ka, p.kd, p.ks, p.shininess
    r.grad_eps = p.grad_eps
    r.out_fp16 = int(bool(out_fp16))
    return r


class Model:
    """An MFA model resident on the current CUDA device (mfa_model_create)."""

    def __init__(self, degree, knots, ctrl, stream=None, layout: str = "auto"):
        import torch
        if np.isscalar(degree):
            degree = (int(degree),) * 3
        self._h = C.c_void_p(0)
        L = lib()
        deg = (C.c_int32 * 3)(*[int(x) for x in degree])
        if isinstance(ctrl, torch.Tensor):
            assert ctrl.dim() == 3
            nw, nv, nu = ctrl.shape
            on_dev = int(ctrl.is_cuda)
            ctrl_c = ctrl.contiguous().float()
            cptr = C.c_void_p(ctrl_c.data_ptr())
        else:
            ctrl_c = np.ascontiguousarray(ctrl, dtype=np.float32)
            nw, nv, nu = ctrl_c.shape
            on_dev = 0
            cptr = C.c_void_p(ctrl_c.ctypes.data)
        n = (C.c_int64 * 3)(nu, nv, nw)
        self._knots = [np.ascontiguousarray(k, dtype=np.float64) for k in knots]
        kp = (C.POINTER(C.c_double) * 3)(*[k.ctypes.data_as(C.POINTER(C.c_double)) for k in self._knots])
        h = C.c_void_p(0)
        opt = ModelOptions_t(LAYOUTS[layout])
        _check(L.mfa_model_create_ex(deg, n, kp, cptr, on_dev, C.byref(opt), _stream_ptr(stream), C.byref(h)))
        self._h = h
        self.degree = tuple(int(x) for x in degree)
        self.nctrl = (nu, nv, nw)

    @classmethod
    def from_workload(cls, w, stream=None, layout: str = "auto"):
        return cls(w.degree, w.knots, w.ctrl, stream=stream, layout=layout)

    @property
    def handle(self):
        return self._h

    def info(self) -> dict:
        d = ModelDesc_t()
        _check(lib().mfa_model_info(self._h, C.byref(d)))
        return dict(degree=tuple(d.degree), nctrl=tuple(d.nctrl), uniform=tuple(d.uniform),
                    v_min=d.v_min, v_max=d.v_max, device_bytes=d.device_bytes, device=d.device,
                    layout={1: "quads", 2: "bezier", 3: "bricks", 4: "bezier_grouped"}.get(d.layout, d.layout), model_bytes=d.model_bytes,
                    create_ms=d.create_ms)

    def close(self):
        if self._h and self._h.value:
            lib().mfa_model_destroy(self._h)
            self._h = C.c_void_p(0)

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # -- queryValueMFA / queryGradientMFA (mfa_eval_batch) --------------------
    def eval(self, u, v, w, grad=True, out=None, n_domain_errors=None, stream=None, binned="auto"):
        """u, v, w: CUDA fp32 tensors (n,).  Returns (value, du, dv, dw)
        (parameter-space partials), or (value,) if grad is False.
        binned: "auto" = the north_star call mfa_eval_batch (large batches are
        binned with stream-ordered scratch from the device pool); True =
        mfa_eval_batch_ws with a workspace from torch's allocator; False =
        mfa_eval_batch_ws without a workspace (the unbinned kernel)."""
        import torch
        n = u.numel()
        dev = u.device
        if out is None:
            out = tuple(torch.empty(n, device=dev, dtype=torch.float32) for _ in range(4 if grad else 1))
        val = out[0]
        du, dv, dw = (out[1], out[2], out[3]) if grad else (None, None, None)
        if binned == "auto":
            _check(lib().mfa_eval_batch(self._h, n, _ptr(u), _ptr(v), _ptr(w), _ptr(val), _ptr(du), _ptr(dv),
                                        _ptr(dw), _ptr(n_domain_errors), _stream_ptr(stream)))
            return out
        ws, nb = None, 0
        if binned and n >= (1 << 16):
            nb = int(lib().mfa_eval_workspace_bytes(self._h, n))
            ws = torch.empty(nb, dtype=torch.uint8, device=dev)   # stream-ordered by torch's allocator
        _check(lib().mfa_eval_batch_ws(self._h, n, _ptr(u), _ptr(v), _ptr(w), _ptr(val), _ptr(du), _ptr(dv),
                                       _ptr(dw), _ptr(n_domain_errors), _ptr(ws), nb, _stream_ptr(stream)))
        return out

    def eval_hessian(self, u, v, w, n_domain_errors=None, stream=None, binned="auto"):
        """NEXT-4 (mfa_eval_hessian): returns (value [n], grad [3,n], hess [6,n]),
        hess rows = d2/du2, d2/dv2, d2/dw2, d2/dudv, d2/dudw, d2/dvdw (parameter space).
        binned: as eval ("auto" = mfa_eval_hessian, False = the unbinned kernel)."""
        import torch
        n = u.numel()
        val = torch.empty(n, device=u.device, dtype=torch.float32)
        grad = torch.empty((3, n), device=u.device, dtype=torch.float32)
        hess = torch.empty((6, n), device=u.device, dtype=torch.float32)
        if binned == "auto":
            _check(lib().mfa_eval_hessian(self._h, n, _ptr(u), _ptr(v), _ptr(w), _ptr(val), _ptr(grad), _ptr(hess),
                                          _ptr(n_domain_errors), _stream_ptr(stream)))
            return val, grad, hess
        ws, nb = None, 0
        if binned and n >= (1 << 16):
            nb = int(lib().mfa_hessian_workspace_bytes(self._h, n))
            ws = torch.empty(nb, dtype=torch.uint8, device=u.device)
        _check(lib().mfa_eval_hessian_ws(self._h, n, _ptr(u), _ptr(v), _ptr(w), _ptr(val), _ptr(grad),
                                         _ptr(hess), _ptr(n_domain_errors), _ptr(ws), nb, _stream_ptr(stream)))
        return val, grad, hess

    # -- Algorithm 1 (mfa_render) ---------------------------------------------
    def render(self, cams, tf, v_lo, v_hi, params, tiles=None, out=None, samples=None, out_fp16=False,
               stream=None, field=None, lights=None, scatter=False, curvature=None):
        """cams: list of Camera; tf: CUDA fp32 tensor (n,4); params: RenderParams.
        field: optional workloads.AnalyticField -- samples take their value
        and/or gradient from the analytic function (mfa_render_field; the
        ground-truth image when both come from it).  lights: optional
        [(direction towards the light, intensity), ...] replacing the
        headlight (mfa_render_ex).  scatter (with tiles): store each pixel at
        its image position in out ([V,H,W,4], possibly a peer GPU's image)
        instead of a packed tile buffer.  curvature: optional (CUDA fp32
        table [n, n, 4] indexed [kappa_2][kappa_1], range) -- the curvature
        transfer function of mfa_render_ex.
        Returns the image [V,H,W,4] (or packed tiles [T,16,16,4] if tiles given)."""
        import torch
        tf = tf.contiguous()
        tft = TF_t(C.c_void_p(tf.data_ptr()), tf.shape[0], float(v_lo), float(v_hi))
        ca = cameras_t(cams)
        pr = params_t(params, out_fp16)
        dt = torch.float16 if out_fp16 else torch.float32
        W, H = cams[0].width, cams[0].height
        tl = None
        if tiles is not None:
            tl = Tiles_t(tiles.shape[0], C.c_void_p(tiles.data_ptr()), int(bool(scatter)))
            shape = (len(cams), H, W, 4) if scatter else (tiles.shape[0], TILE, TILE, 4)
        else:
            shape = (len(cams), H, W, 4)
        if out is None:
            out = torch.empty(shape, device=tf.device, dtype=dt)
        ext = None
        if field is not None or lights or curvature is not None:
            ft = field_t(field) if field is not None else None
            ld = np.ascontiguousarray([l[0] for l in lights or []], dtype=np.float64).reshape(-1)
            li = np.ascontiguousarray([l[1] for l in lights or []], dtype=np.float64)
            ctab, crange = (curvature[0].contiguous(), float(curvature[1])) if curvature is not None else (None, 0.0)
            ext = RenderExt_t(C.pointer(ft) if ft is not None else None, len(lights or []),
                              ld.ctypes.data_as(C.POINTER(C.c_double)), li.ctypes.data_as(C.POINTER(C.c_double)),
                              C.c_void_p(ctab.data_ptr()) if ctab is not None else None,
                              ctab.shape[0] if ctab is not None else 0, crange)
        _check(lib().mfa_render_ex(self._h, len(cams), ca, C.byref(tft), C.byref(pr),
                                   C.byref(ext) if ext is not None else None,
                                   C.byref(tl) if tl is not None else None, _ptr(out), _ptr(samples),
                                   _stream_ptr(stream)))
        return out

    def render_host(self, cams, tf_host: np.ndarray, v_lo, v_hi, params, out_host, out_fp16=False,
                    stream=None) -> int:
        """Host-buffer render (mfa_render_host): tf from host memory, image
        written to out_host (pinned CPU tensor [V,H,W,4]).  Returns the
        composited-sample count."""
        tfh = np.ascontiguousarray(tf_host, dtype=np.float32)
        cnt = C.c_ulonglong(0)
        _check(lib().mfa_render_host(self._h, len(cams), cameras_t(cams), C.c_void_p(tfh.ctypes.data),
                                     tfh.shape[0], float(v_lo), float(v_hi), C.byref(params_t(params, out_fp16)),
                                     C.c_void_p(out_host.data_ptr()), C.byref(cnt), _stream_ptr(stream)))
        return int(cnt.value)


def _render_host_views(self, cams, tf_host: np.ndarray, v_lo, v_hi, params, view_ptrs, out_fp16=False,
                       stream=None) -> int:
    """mfa_render_host_views: view v of cams goes to host address view_ptrs[v]
    ([H,W,4] fp32 or fp16, page-locked).  Returns the composited-sample count."""
    tfh = np.ascontiguousarray(tf_host, dtype=np.float32)
    cnt = C.c_ulonglong(0)
    ptrs = (C.c_void_p * len(cams))(*[int(x) for x in view_ptrs])
    _check(lib().mfa_render_host_views(self._h, len(cams), cameras_t(cams), C.c_void_p(tfh.ctypes.data),
                                       tfh.shape[0], float(v_lo), float(v_hi), C.byref(params_t(params, out_fp16)),
                                       ptrs, C.byref(cnt), _stream_ptr(stream)))
    return int(cnt.value)


Model.render_host_views = _render_host_views


class IpcBuffer:
    """A device buffer allocated by libmfa (mfa_ipc_alloc: cudaMalloc on the
    current device) together with its CUDA IPC handle, so another process can
    map it (mfa_ipc_open) -- the multi-GPU direct-store image.  tensor(shape,
    dtype) views it as a torch tensor (zero copy, __cuda_array_interface__)."""

    def __init__(self, nbytes: int):
        ptr = C.c_void_p(0)
        h = C.create_string_buffer(64)
        _check(lib().mfa_ipc_alloc(int(nbytes), C.byref(ptr), h))
        self.ptr = ptr.value
        self.nbytes = int(nbytes)
        self.handle = h.raw[:64]

    def tensor(self, shape, dtype):
        import torch
        typestr = {torch.float32: "<f4", torch.float16: "<f2", torch.uint8: "|u1"}[dtype]
        buf = self

        class _View:
            __cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (buf.ptr, False),
                                        "version": 3, "strides": None}
        t = torch.as_tensor(_View(), device="cuda")
        t._mfa_owner = self   # keep the allocation alive with the tensor
        return t

    def close(self):
        if self.ptr:
            _check(lib().mfa_ipc_free(C.c_void_p(self.ptr)))
            self.ptr = 0

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def unpack_tiles(packed, tiles, n_views, width, height, out=None, stream=None):
    """Scatter packed [T,16,16,4] tiles into [V,H,W,4] fp32 images (mfa_unpack_tiles)."""
    import torch
    if out is None:
        out = torch.zeros((n_views, height, width, 4), device=packed.device, dtype=torch.float32)
    _check(lib().mfa_unpack_tiles(_ptr(packed), int(packed.dtype == torch.float16), _ptr(tiles), tiles.shape[0],
                                  n_views, width, height, _ptr(out), _stream_ptr(stream)))
    return out


def image_quality(a, b, err_map=False, workspace=None, stream=None):
    """MSE / PSNR / SSIM of image a against b (mfa_image_quality): CUDA fp32
    tensors [H,W,4] (premultiplied RGBA; alpha ignored).  Returns a dict with
    "mse", "psnr", "ssim" (and "err_map", an [H,W] tensor, if requested)."""
    import torch
    assert a.shape == b.shape and a.dim() == 3 and a.shape[2] == 4
    a, b = a.contiguous().float(), b.contiguous().float()
    H, W = a.shape[0], a.shape[1]
    nbytes = int(lib().mfa_image_quality_workspace(W, H))
    if workspace is None or workspace.numel() < nbytes:
        workspace = torch.empty(max(nbytes, 1), dtype=torch.uint8, device=a.device)
    out = torch.empty(3, dtype=torch.float64, device=a.device)
    em = torch.empty((H, W), dtype=torch.float32, device=a.device) if err_map else None
    _check(lib().mfa_image_quality(W, H, _ptr(a), _ptr(b), _ptr(em), _ptr(workspace), nbytes, _ptr(out),
                                   _stream_ptr(stream)))
    r = out.cpu().tolist()
    res = {"mse": r[0], "psnr": r[1], "ssim": r[2]}
    if err_map:
        res["err_map"] = em
    return res


def _knots_arg(knots):
    ks = [np.ascontiguousarray(k, dtype=np.float64) for k in knots]
    arr = (C.POINTER(C.c_double) * 3)(*[k.ctypes.data_as(C.POINTER(C.c_double)) for k in ks])
    return ks, arr


def fit_grid(values, degree: int, knots, want64=False, stream=None):
    """NEXT-3 least-squares fit (mfa_fit_grid): values = CUDA fp32 grid
    [m_w, m_v, m_u]; knots = 3 fp64 clamped knot vectors.  Returns the control
    values [n_w, n_v, n_u] (fp32, plus the fp64 copy if want64)."""
    import torch
    values = values.contiguous()
    mw, mv, mu = values.shape
    dims = (C.c_int64 * 3)(mu, mv, mw)
    n = [len(k) - degree - 1 for k in knots]
    nct = (C.c_int64 * 3)(*n)
    ks, karr = _knots_arg(knots)
    c32 = torch.empty((n[2], n[1], n[0]), dtype=torch.float32, device=values.device)
    c64 = torch.empty((n[2], n[1], n[0]), dtype=torch.float64, device=values.device) if want64 else None
    _check(lib().mfa_fit_grid(dims, _ptr(values), int(degree), nct, karr, _ptr(c32), _ptr(c64), _stream_ptr(stream)))
    return (c32, c64) if want64 else c32


def encode_grid(values, degree: int, nctrl_init, e_max: float, max_rounds: int, max_ctrl, stream=None):
    """NEXT-3 adaptive encoder (mfa_encode_grid).  Returns (knots [3 x np.ndarray],
    ctrl CUDA fp32 [n_w, n_v, n_u], result dict, per-round log (rounds x 5))."""
    import torch
    values = values.contiguous()
    mw, mv, mu = values.shape
    dims = (C.c_int64 * 3)(mu, mv, mw)
    cfg = EncodeConfig_t(int(degree), (C.c_int64 * 3)(*nctrl_init), float(e_max), int(max_rounds),
                         (C.c_int64 * 3)(*max_ctrl))
    cap = [min(int(max_ctrl[d]), (mu, mv, mw)[d]) for d in range(3)]
    kbuf = [np.zeros(cap[d] + degree + 1) for d in range(3)]
    _, karr = _knots_arg(kbuf)
    ctrl = torch.empty(cap[0] * cap[1] * cap[2], dtype=torch.float32, device=values.device)
    res = EncodeResult_t()
    log = np.zeros((max_rounds + 1, 5))
    _check(lib().mfa_encode_grid(dims, _ptr(values), C.byref(cfg), karr, _ptr(ctrl), C.byref(res),
                                 C.c_void_p(log.ctypes.data), _stream_ptr(stream)))
    n = [int(x) for x in res.nctrl]
    knots = [kbuf[d][:n[d] + degree + 1].copy() for d in range(3)]
    out = dict(nctrl=tuple(n), rounds=res.rounds, converged=bool(res.converged), max_err=res.max_err,
               rms_err=res.rms_err)
    return knots, ctrl[:n[0] * n[1] * n[2]].view(n[2], n[1], n[0]), out, log[:res.rounds].copy()


def enable_peer_access(peer_device: int):
    """Let kernels on the current device access memory of peer_device
    (mfa_enable_peer_access; no-op if already enabled or the same device)."""
    _check(lib().mfa_enable_peer_access(int(peer_device)))


class PeerBuffer:
    """A device buffer of another process mapped on the current device
    (mfa_ipc_open): data_ptr() for the entry points, shape / dtype for the
    caller; close() unmaps it."""

    _open = {}   # handle -> [base, users]: an allocation is mapped once per process

    def __init__(self, handle: bytes, offset: int, shape, dtype):
        self._handle = bytes(handle)
        ent = PeerBuffer._open.get(self._handle)
        if ent is None:
            base = C.c_void_p(0)
            _check(lib().mfa_ipc_open(self._handle, C.byref(base)))
            ent = PeerBuffer._open[self._handle] = [base.value, 0]
        ent[1] += 1
        self._base = ent[0]
        self._ptr = ent[0] + int(offset)
        self.shape = tuple(shape)
        self.dtype = dtype

    def data_ptr(self) -> int:
        return self._ptr

    def close(self):
        if self._base:
            ent = PeerBuffer._open[self._handle]
            ent[1] -= 1
            if ent[1] == 0:
                del PeerBuffer._open[self._handle]
                _check(lib().mfa_ipc_close(C.c_void_p(self._base)))
            self._base = self._ptr = 0


def version() -> str:
    return lib().mfa_version().decode()


def probe_fp32(mode: str = "ffma2") -> float:
    """Measured FP32 FMA throughput (TFLOP/s) on the current device (K5)."""
    v = C.c_double(0)
    _check(lib().mfa_probe_fp32({"ffma": 0, "ffma2": 1, "ffma_imm": 2}[mode], C.byref(v)))
    return v.value


def probe_read_bw(nbytes: int, reps: int = 20) -> float:
    """Measured read bandwidth (GB/s) of an nbytes buffer read reps times (K5)."""
    v = C.c_double(0)
    _check(lib().mfa_probe_read_bw(int(nbytes), int(reps), C.byref(v)))
    return v.value
