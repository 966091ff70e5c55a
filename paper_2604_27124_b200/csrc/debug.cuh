// debug.cuh -- timing-experiment switches, DEBUG BUILDS ONLY.
//
// Each SIGATTN_DBG_* switch removes work from a kernel (so its results are WRONG) to measure where
// the time goes; build.build_variant() compiles them into separate
// libsigattn_<name>.so files with -DSIGATTN_DEBUG_BUILD.  A release build that sets any of them
// does not compile.
#pragma once

#ifndef SIGATTN_DBG_FWD_NOSIGMA
#define SIGATTN_DBG_FWD_NOSIGMA 0   // forward: P = bits of S, no sigma work
#endif
#ifndef SIGATTN_DBG_FWD_NOTMA_KV
#define SIGATTN_DBG_FWD_NOTMA_KV 0  // forward: K/V tiles loaded once per ring slot, then reused (stale)
#endif
#ifndef SIGATTN_DBG_NOCOMPUTE
#define SIGATTN_DBG_NOCOMPUTE 0     // backward: compute warps skip sigma + TMEM I/O
#endif
#ifndef SIGATTN_DBG_EPI_NOLD
#define SIGATTN_DBG_EPI_NOLD 0      // backward: epilogue skips TMEM loads and global writes
#endif
#ifndef SIGATTN_DBG_NORED
#define SIGATTN_DBG_NORED 0         // backward: no dQ reduce-add into global memory
#endif
#ifndef SIGATTN_DBG_NOTMA_QDO
#define SIGATTN_DBG_NOTMA_QDO 0     // backward: Q/dO tiles loaded once, then reused (stale)
#endif
#ifndef SIGATTN_DBG_MMAONLY
#define SIGATTN_DBG_MMAONLY 0       // backward: MMA + TMA pipeline alone (no compute / epilogue waits)
#endif
#ifndef SIGATTN_DBG_EPI_NOSTORE
#define SIGATTN_DBG_EPI_NOSTORE 0   // two-tile forward: the O epilogue skips its global stores
#endif
#ifndef SIGATTN_DBG_NOFILL
#define SIGATTN_DBG_NOFILL 0        // fwd / bwd: skip the padded-row zero fills (outputs incomplete)
#endif

#if !defined(SIGATTN_DEBUG_BUILD) &&                                                                     \
    (SIGATTN_DBG_FWD_NOSIGMA || SIGATTN_DBG_FWD_NOTMA_KV || SIGATTN_DBG_NOCOMPUTE || SIGATTN_DBG_EPI_NOLD || \
     SIGATTN_DBG_NORED || SIGATTN_DBG_NOTMA_QDO || SIGATTN_DBG_MMAONLY || SIGATTN_DBG_NOFILL || SIGATTN_DBG_EPI_NOSTORE)
#error "SIGATTN_DBG_* switches make the kernels compute wrong results: timing builds only (-DSIGATTN_DEBUG_BUILD)"
#endif
