// decoder_common.cuh -- device helpers shared by the decoders (K1 / K1b in kernels.cu, K1q in
// kernels_q.cu): group shuffles, (ready, job) heads, gene-row staging.
#pragma once

#include <cuda_pipeline.h>

#include "launch.h"

namespace ffsga_dev {
namespace {

// ---- checked build (python build.py --checked, -DFFSGA_CHECKED): device-side bounds and
// invariant checks standing in for compute-sanitizer (closed on this GPU pool).  The first
// failed check is kept as code << 48 | a << 24 | b and read by ffsga_cuda_checked_status();
// kernels continue (indices stay in range), so a failure never hangs or faults the device.
#ifdef FFSGA_CHECKED
__device__ unsigned long long g_check_fail;
__device__ __forceinline__ void check_fail(unsigned code, unsigned a, unsigned b) {
    atomicCAS(&g_check_fail, 0ull,
              ((unsigned long long)code << 48) | ((unsigned long long)(a & 0xFFFFFFu) << 24) | (b & 0xFFFFFFu));
}
#define FFSGA_CHECK(cond, code, a, b)                                  \
    do {                                                               \
        if (!(cond)) check_fail((code), (unsigned)(a), (unsigned)(b)); \
    } while (0)
#else
#define FFSGA_CHECK(cond, code, a, b) \
    do {                              \
    } while (0)
#endif

constexpr unsigned kFull = 0xffffffffu;
constexpr unsigned long long kNoErr = ~0ull;

__device__ __forceinline__ double dinf() { return __longlong_as_double(0x7FF0000000000000LL); }

template <int G>
__device__ __forceinline__ double group_max(double v) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        double o = __shfl_xor_sync(kFull, v, off, G);
        v = (v < o) ? o : v;
    }
    return v;
}

template <int G>
__device__ __forceinline__ int group_min_int(int v) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) v = min(v, __shfl_xor_sync(kFull, v, off, G));
    return v;
}

template <int G>
__device__ __forceinline__ void group_min_key(double& c, int& j) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        double oc = __shfl_xor_sync(kFull, c, off, G);
        int oj = __shfl_xor_sync(kFull, j, off, G);
        if (oc < c || (oc == c && oj < j)) { c = oc; j = oj; }
    }
}


__device__ __forceinline__ bool key_lt(double va, int ja, double vb, int jb) {  // (ready, job) order
    return (va < vb) | ((va == vb) & (ja < jb));
}

// The NS list heads of a lane are kept sorted by (ready, job), so the next job to dispatch is
// always head 0.  After a pop, the successor from the same list is inserted in one step: all
// NS-1 comparisons are independent and each slot is rebuilt with two selects, so the
// loop-carried dependency is one compare and two selects deep (not a log2(NS) tournament).
template <int NS>
__device__ __forceinline__ void heads_sort(double (&v)[NS], int (&j)[NS]) {
#pragma unroll
    for (int i = 0; i < NS; ++i) {
#pragma unroll
        for (int k = NS - 1; k > i; --k) {
            const bool sw = key_lt(v[k], j[k], v[k - 1], j[k - 1]);
            const double v0 = v[k - 1], v1 = v[k];
            const int j0 = j[k - 1], j1 = j[k];
            v[k - 1] = sw ? v1 : v0;
            v[k] = sw ? v0 : v1;
            j[k - 1] = sw ? j1 : j0;
            j[k] = sw ? j0 : j1;
        }
    }
}

// EXACT: (ready, job) order.  Otherwise ready times only (one compare per head instead of
// three); equal ready times then pop back to back in some order, which stage_pass detects, and
// the chromosome is decoded again with the exact order (never for continuous processing times).
template <int NS, bool EXACT>
__device__ __forceinline__ void heads_replace_min(double (&v)[NS], int (&j)[NS], double x, int xj) {
    bool c[NS];
#pragma unroll
    for (int k = 0; k + 1 < NS; ++k) c[k] = EXACT ? key_lt(v[k + 1], j[k + 1], x, xj) : (v[k + 1] < x);
    double nv[NS];
    int nj[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const bool after = (k + 1 < NS) ? c[k] : false;  // slot k takes head k+1
        const bool here = (k == 0) ? true : c[k - 1];    // else slot k takes x if x belongs at k
        const double keep = here ? x : v[k];
        const int keepj = here ? xj : j[k];
        nv[k] = after ? v[(k + 1 < NS) ? k + 1 : k] : keep;
        nj[k] = after ? j[(k + 1 < NS) ? k + 1 : k] : keepj;
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        v[k] = nv[k];
        j[k] = nj[k];
    }
}


// ---- packed heads (K1's ready-only pass when DevInst::pk_bits > 0).  key = the ready time's
// bits with the low pk_bits replaced by the job id.  For sign-clear finite ready times one fp64
// compare of two keys orders them by (ready truncated above those bits, job): the exact
// (ready, job) order except between ready times that agree above the job bits, which stage_pass
// flags like a tie (exact re-decode).  The dropped bits of job j's ready time wait in a u16 array
// (the link region, indexed by job) until j is popped.
__device__ __forceinline__ double pk_pack(double v, int j, unsigned mask) {
    return __hiloint2double(__double2hiint(v), (int)(((unsigned)__double2loint(v) & ~mask) | (unsigned)j));
}
__device__ __forceinline__ int pk_job(double k, unsigned mask) { return (int)((unsigned)__double2loint(k) & mask); }
__device__ __forceinline__ unsigned pk_low(double v, unsigned mask) { return (unsigned)__double2loint(v) & mask; }
__device__ __forceinline__ double pk_value(double k, unsigned low, unsigned mask) {
    return __hiloint2double(__double2hiint(k), (int)(((unsigned)__double2loint(k) & ~mask) | low));
}
// above every real key (ready times < 1e300), job field END
__device__ __forceinline__ double pk_sentinel(int end, unsigned mask) {
    return __hiloint2double(0x7FEFFFFF, (int)((0xFFFFFFFFu & ~mask) | (unsigned)end));
}
// zero iff two keys / ready times agree above the job bits (two LOP3s)
__device__ __forceinline__ unsigned pk_high_diff(double a, double b, unsigned mask) {
    return ((unsigned)__double2hiint(a) ^ (unsigned)__double2hiint(b)) |
           (((unsigned)__double2loint(a) ^ (unsigned)__double2loint(b)) & ~mask);
}

template <int NS>
__device__ __forceinline__ void heads_sort_pk(double (&v)[NS]) {
#pragma unroll
    for (int i = 0; i < NS; ++i) {
#pragma unroll
        for (int k = NS - 1; k > i; --k) {
            const double v0 = v[k - 1], v1 = v[k];
            const bool sw = v1 < v0;
            v[k - 1] = sw ? v1 : v0;
            v[k] = sw ? v0 : v1;
        }
    }
}

// heads_replace_min on keys alone: two selects per 32-bit half per slot, no job ids
template <int NS>
__device__ __forceinline__ void heads_replace_min_pk(double (&v)[NS], double x) {
    bool c[NS];
#pragma unroll
    for (int k = 0; k + 1 < NS; ++k) c[k] = v[k + 1] < x;
    double nv[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const bool after = (k + 1 < NS) ? c[k] : false;
        const bool here = (k == 0) ? true : c[k - 1];
        const double keep = here ? x : v[k];
        nv[k] = after ? v[(k + 1 < NS) ? k + 1 : k] : keep;
    }
#pragma unroll
    for (int k = 0; k < NS; ++k) v[k] = nv[k];
}


__device__ __forceinline__ void stage_barrier(bool cta) {
    if (cta)
        __syncthreads();
    else
        __syncwarp();
}


// Asynchronous copy of gene row s into `row` (cp.async, 16 B per request, L1 bypass).
template <int G>
__device__ __forceinline__ void prefetch_row(const DevInst& I, const uint8_t* genes, int s, int m, uint8_t* row) {
    const uint8_t* src = genes + (size_t)s * I.Jpad;
    for (int v = m; v < I.Jpad / 16; v += G) __pipeline_memcpy_async(row + 16 * v, src + 16 * v, 16);
    __pipeline_commit();
}

// Group-uniform: does the staged row hold a gene >= Mlimit (model.cpp:81-83)?  Every lane of
// the warp must call it (the reduction shuffles).
template <int G>
__device__ __forceinline__ bool row_has_bad(const DevInst& I, const uint8_t* row, int m, int Mlimit, bool doit) {
    unsigned bad = 0;
    if (doit) {
        const unsigned lim = 0x01010101u * (unsigned)min(Mlimit, 255);
        const uint4* v4 = reinterpret_cast<const uint4*>(row);
        for (int v = m; v < I.Jpad / 16; v += G) {
            const uint4 x = v4[v];
            bad |= __vcmpgeu4(x.x, lim) | __vcmpgeu4(x.y, lim) | __vcmpgeu4(x.z, lim) | __vcmpgeu4(x.w, lim);
        }
    }
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) bad |= __shfl_xor_sync(kFull, bad, off, G);
    return bad != 0;
}


template <int G>
__device__ __forceinline__ double group_min_d(double v) {
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        double o = __shfl_xor_sync(kFull, v, off, G);
        v = (o < v) ? o : v;
    }
    return v;
}


}  // namespace
}  // namespace ffsga_dev
