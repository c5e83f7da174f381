/*
 * memascend/state_pool.h — C entry points of the drop-in C++ Pool
 * (include/memascend/pool.hpp) for the streamed optimizer state of configs[3]
 * (north star item (1): "the adaptive, alignment-free pinned buffer pool,
 * which becomes one cudaHostRegister'd pool whose sub-group slices are staged
 * H2D/D2H").  Exported by libmemascend.so, for trainers that are not C++
 * (the Python bench binds it with ctypes).
 *
 * A state pool is a memascend::Pool in adaptive mode over the inventory
 * "master.g<k>", "m.g<k>", "v.g<k>" (fp32, one exact-fit slot class per
 * distinct sub-group size, pool.cpp:22-68) whose backing comes from the
 * registering PinnedAllocator (alignment-free policy); every tensor is
 * checked out for the pool's lifetime and handed out as its host span and
 * its device_span (the same bytes through UVA), ready for
 * ma_stepper_apply_streamed.
 */
#ifndef MEMASCEND_STATE_POOL_H
#define MEMASCEND_STATE_POOL_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct memascend_state_pool memascend_state_pool;

/* n_params elements split into sub-groups of `subgroup` (the last shorter).
 * Status codes are MA_* (include/memascend_b200.h); memascend_last_error()
 * describes a failure. */
int memascend_state_pool_create(uint64_t n_params, uint64_t subgroup, memascend_state_pool** out);
/* which: 0 = master (p), 1 = m, 2 = v. */
int memascend_state_pool_tensor(memascend_state_pool* p, uint64_t group, int which, void** host,
                                void** device, uint64_t* elems);
/* Pool::stats(): slot payload capacity, backing bytes, live (checked-out)
 * bytes, checkouts; classes = number of slot classes. */
int memascend_state_pool_stats(memascend_state_pool* p, uint64_t* capacity_bytes,
                               uint64_t* backing_bytes, uint64_t* live_bytes,
                               uint64_t* checkouts, uint64_t* classes);
int memascend_state_pool_destroy(memascend_state_pool* p);
const char* memascend_last_error(void);

#ifdef __cplusplus
}
#endif

#endif
