/* salvox_bench.h -- measurement entry points of libsalvox_b200 (not part of the
 * reference API; used by bench.py for the live roofline). */
#ifndef SALVOX_BENCH_H
#define SALVOX_BENCH_H

#include "salvox_capi.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Peak rate of kb_kernel's inner-loop pair (u8 bin fetch from a shared tile at
 * a warp-uniform offset + one ATOMS.ADD into a lane-private column), measured
 * by a microkernel with the identical instruction mix and occupancy:
 * *atoms_updates_per_s (the exhaustive roofline denominator),
 * *lds_fetches_per_s (bin fetches alone, no histogram update) and
 * *atoms_only_per_s (ATOMS.ADD alone with register-resident bins: the
 * one-atomic-per-update floor of any shared-memory histogram design). */
SALVOX_API int salvox_probe_smem_peak(salvox_ctx* ctx, int iters, double* atoms_updates_per_s,
                                      double* lds_fetches_per_s, double* atoms_only_per_s);
/* Of the last salvox_probe_smem_peak call: the ATOMS rate of kb_quad_kernel's
 * walk with its bin-word loads removed (PRMT-built addresses, panel in the
 * immediate, 8 warps x 4 columns); it is one of the layouts whose best is
 * *atoms_only_per_s. */
SALVOX_API double salvox_probe_prmt_rate(void);

/* Times every exhaustive kb_kernel launch with CUDA events on the launching
 * stream while on (resets the accumulators). */
SALVOX_API int salvox_ctx_set_profiling(salvox_ctx* ctx, int on);
/* Accumulated kb_kernel time (ms), launch count and algorithmic histogram
 * updates (computed voxels x (|B(R_max)| - 1)) since profiling was enabled. */
SALVOX_API int salvox_ctx_kernel_time(salvox_ctx* ctx, double* kb_ms_total, int64_t* kb_launches,
                                      double* kb_updates_total);

#ifdef __cplusplus
}
#endif
#endif
