// tmem.cuh -- Tensor Memory (TMEM) as per-thread persistent storage (sm_100a).
//
// The resident decoder keeps each check row's compact state (A_m, B_m, ñ_m, s_mn;
// PAPER.md P:335 "persistent data stored in memory") in TMEM: thread t of warp w
// owns TMEM lane 32*(w%4) + (t%32) and a private range of columns, so a row's
// state never travels to L2/HBM between iterations.  Accesses are tcgen05.ld /
// tcgen05.st (SASS LDTM / STTM) with the 32x32b shape: each thread reads/writes
// its own lane.  Allocation is done once per CTA by warp 0 (tcgen05.alloc +
// relinquish_alloc_permit), freed by the same warp at exit.
#pragma once
#include <cstdint>

namespace ldpc {

__device__ __forceinline__ uint32_t tmem_alloc_cta(uint32_t *slot, uint32_t ncols) {
    if ((threadIdx.x >> 5) == 0) {
        const uint32_t sa = (uint32_t)__cvta_generic_to_shared(slot);
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(sa), "r"(ncols));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
    }
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    return *(volatile uint32_t *)slot;
}

__device__ __forceinline__ void tmem_free_cta(uint32_t base, uint32_t ncols) {
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
    if ((threadIdx.x >> 5) == 0)
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(base), "r"(ncols));
}

// lane-quadrant base address of this warp
__device__ __forceinline__ uint32_t tmem_warp_base(uint32_t base) {
    return base + ((uint32_t)(32 * ((threadIdx.x >> 5) & 3)) << 16);
}

__device__ __forceinline__ void tmem_ld1(uint32_t taddr, uint32_t &a) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(a) : "r"(taddr));
}
__device__ __forceinline__ void tmem_ld2(uint32_t taddr, uint32_t &a, uint32_t &b) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x2.b32 {%0, %1}, [%2];" : "=r"(a), "=r"(b) : "r"(taddr));
}
__device__ __forceinline__ void tmem_st1(uint32_t taddr, uint32_t a) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x1.b32 [%0], {%1};" ::"r"(taddr), "r"(a));
}
__device__ __forceinline__ void tmem_st2(uint32_t taddr, uint32_t a, uint32_t b) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x2.b32 [%0], {%1, %2};" ::"r"(taddr), "r"(a), "r"(b));
}
__device__ __forceinline__ void tmem_ld4(uint32_t taddr, uint32_t &a, uint32_t &b, uint32_t &c, uint32_t &d) {
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "r"(taddr));
}
__device__ __forceinline__ void tmem_st4(uint32_t taddr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1, %2, %3, %4};" ::"r"(taddr), "r"(a), "r"(b), "r"(c),
                 "r"(d));
}
// wait for outstanding tcgen05.ld, tying eight destination registers
__device__ __forceinline__ void tmem_wait_ld_dep8(uint32_t (&v)[8]) {
    asm volatile("tcgen05.wait::ld.sync.aligned;"
                 : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]), "+r"(v[6]), "+r"(v[7])
                 :: "memory");
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }
// wait for outstanding tcgen05.ld of this thread, tying the destination registers so the
// compiler cannot hoist their uses above the wait
__device__ __forceinline__ void tmem_wait_ld_dep(uint32_t &a, uint32_t &b, uint32_t &c) {
    asm volatile("tcgen05.wait::ld.sync.aligned;" : "+r"(a), "+r"(b), "+r"(c)::"memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }

}  // namespace ldpc
