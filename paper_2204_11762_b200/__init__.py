"""B200-native MFA-DVR hot path (arXiv 2204.11762): direct volume ray casting
of a tensor-product B-spline (MFA) model on sm_100a.

    from paper_2204_11762_b200 import Model, workloads
    w = workloads.make_config(3)
    m = Model.from_workload(w)            # mfa_model_create
    val, du, dv, dw = m.eval(u, v, w)     # mfa_eval_batch (CUDA tensors)
    img = m.render(w.cameras, tf, w.v_lo, w.v_hi, w.params)   # mfa_render

The C ABI is include/mfa.h; libmfa.so is built in-tree by
``python -m paper_2204_11762_b200.build``.  There is no CPU fallback.
"""
from ._lib import Model, MfaError, encode_grid, fit_grid, image_quality, lib, unpack_tiles, version  # noqa: F401

__all__ = ["Model", "MfaError", "encode_grid", "fit_grid", "image_quality", "lib", "unpack_tiles", "version"]
