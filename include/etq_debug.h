/*
 * etq_debug.h — measurement / test hooks of libetq that are not part of the product ABI (etq.h).
 */
#ifndef ETQ_DEBUG_H
#define ETQ_DEBUG_H

#include "etq.h"

#ifdef __cplusplus
extern "C" {
#endif

/* Process-wide implementation switches for A/B measurements and tests (NOT for production use:
 * they are global mutable state shared by every problem in the process; the defaults are the
 * measured-best configuration).  Results are identical either way, bitwise unless stated:
 *   option 0 = temporally blocked Chebyshev smoothing on the Stokes interior-stencil levels
 *              (value 1 = on [default], 0 = one kernel per Chebyshev step);
 *   option 1 = coarsest level n that uses it [64] (smaller grids are launch-latency bound);
 *   option 2 = matrix-free Stokes saddle apply (1 [default]) or the stored SELL rows (0);
 *   option 3 = MINRES loop as one CUDA graph with a device-side while node (1 [default]) or one
 *              graph launch and one flag read-back per iteration (0);
 *   option 4 = launch priority of the Chebyshev-SGS pressure kernels (0 = lowest [default], 1 = highest);
 *   option 5 = coarse V-cycle levels (n <= 16) in one CTA with every vector in shared memory and
 *              the class stencils (1 [default], Stokes only) or through the stored rows in global memory (0);
 *   option 6 = matrix-free Stokes saddle apply from shared-memory tiles (1 [default]) or by global
 *              gathers (0); only with option 2 = 1;
 *   option 7 = programmatic dependent launches between the Chebyshev-SGS steps (1 [default]) or plain
 *              stream order (0);
 *   option 8 = programmatic dependent launches between the kernels of the Q2 V-cycle (1 [default]) or
 *              plain stream order (0);
 *   option 9 = nested-Q2 prolongation from shared-memory tiles (1 [default]) or by gathers (0);
 *   option 10 = Chebyshev-SGS on parity planes with TMA windows (1) or the lexicographic tiles (0 [default]);
 *               outputs agree to rounding (the k^T y sum order differs);
 *   option 11 = the leaner temporally blocked smoother k_cheb_tile2 (1 [default], grouped symmetric
 *               stencil sums: agrees to rounding) or k_cheb_tile (0, bitwise the per-step path);
 *   option 12 = k_cheb_tile3, the smoother with the residual in registers (1 [default], bitwise the
 *               k_cheb_tile2 V-cycle) or k_cheb_tile2 (0);
 *   option 13 = programmatic dependent launches inside the V-cycle of P2 (1 [default]) - bitwise the same;
 *   option 14 = matrix-free interior rows of the cavity-wind F levels (1 [default]) or stored SELL rows (0);
 *   option 15 = Chebyshev-SGS y_prev read in the Q pass (1 [default]) or staged by cp.async (0) - bitwise;
 *   option 16 = Chebyshev-SGS window: 0 = automatic [default: 64 x 32, with 512 threads when the tiles
 *               fit one wave], 1 = 64 x 64, 2 = 64 x 32 / 256 threads, 3 = 64 x 32 / 512 threads - bitwise sweeps;
 *   option 17 = programmatic dependent launches between the kernels of the F V-cycle inside the Oseen
 *               preconditioners (1 [default]) or plain launches (0) - bitwise the same;
 *   option 18 = the tiled smoother prefetches into L2 the window of the tile that follows it on its SM
 *               (1 [default]) or not (0) - bitwise the same.
 * Applies to solves whose CUDA graphs are captured afterwards (re-run etq_precond_setup). */
etq_status etq_debug_set_option(int32_t option, int32_t value);

#ifdef __cplusplus
}
#endif
#endif /* ETQ_DEBUG_H */
