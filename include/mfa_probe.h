/*
 * mfa_probe.h -- measurement probes for the roofline (kernel K5).
 *
 * The north_star roofline of the render path is the lesser of
 *   FP32 FMA peak / counted FLOPs per sample   and
 *   L2 bandwidth  / counted control-point bytes per sample.
 * Neither peak is in MEASURED_PEAKS.json, so these calls measure them on the
 * current device (synchronously; CUDA events; a few hundred ms each).
 */
#ifndef MFA_PROBE_H
#define MFA_PROBE_H

#include <stdint.h>

#include "mfa.h"

#ifdef __cplusplus
extern "C" {
#endif

/* FP32 throughput of independent FMA chains on every SM, in TFLOP/s (FMA = 2).
 * mode 0: FFMA with three register operands; 1: FFMA2 (packed pairs);
 * 2: FFMA with an immediate operand. */
mfa_status mfa_probe_fp32(int32_t mode, double* tflops);

/* Read bandwidth in GB/s of `bytes` (multiple of 4096) read `reps` times by
 * all SMs with 16-byte loads that bypass L1 (ld.global.cg).  bytes well below
 * the L2 size measures L2 bandwidth; well above it, HBM. */
mfa_status mfa_probe_read_bw(int64_t bytes, int32_t reps, double* gbps);

#ifdef __cplusplus
}
#endif
#endif /* MFA_PROBE_H */
