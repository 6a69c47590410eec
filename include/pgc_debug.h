/*
 * pgc_debug.h -- diagnostics of the JP-ADG library (not needed by users).
 *
 * pgc_debug_set_trace: when `t_grab` and `t_done` are non-NULL DEVICE arrays
 * of n uint64 entries, the next calls on this thread record, for every vertex
 * v, the %globaltimer value (ns) at which a JP worker took v (t_grab[v]) and
 * stored its color (t_done[v]).  Pass NULLs to switch tracing off.  The
 * pointers are only used by calls whose graph has exactly `n` vertices.
 * Returns PGC_OK, or PGC_EINVAL if only one pointer is NULL or n < 0.
 */
#ifndef PGC_DEBUG_H
#define PGC_DEBUG_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

int pgc_debug_set_trace(uint64_t* t_grab, uint64_t* t_done, int64_t n);

#ifdef __cplusplus
}
#endif

#endif /* PGC_DEBUG_H */
