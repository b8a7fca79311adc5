// Device helpers shared by the library's translation units (kernels.cu; repair.cu, which
// is compiled as relocatable device code for its device-side launch).  Internal.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include "lmsgd_internal.h"

namespace lmsgd {

// Programmatic dependent launch (sm_90+): every product kernel lets the next kernel
// in the stream be scheduled immediately and waits for its own predecessors to
// complete (and their memory to be visible) before touching any data.  This hides
// the launch latency between the step's kernels without changing their ordering.
__device__ __forceinline__ void pdl_enter() {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

__device__ __forceinline__ uint64_t globaltimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// `last` record in the public lmsgd_step_status layout:
// {int64 first (-1 none), int64 pack_sat, int64 sum_sat, int32 skipped, int32 error}
__device__ __forceinline__ void store_last(int64_t* last, int64_t first, int64_t psat, int64_t ssat,
                                           int64_t err, int64_t skipped) {
    last[0] = first == kNone ? -1 : first;
    last[1] = psat;
    last[2] = ssat;
    int32_t* tail = reinterpret_cast<int32_t*>(last + 3);
    tail[0] = (int32_t)skipped;
    tail[1] = (int32_t)(err ? err : (first != kNone ? (int64_t)LMSGD_ERR_NONFINITE : 0));
}

}  // namespace lmsgd
