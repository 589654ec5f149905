// device.cuh -- device-side data layout, SplitMix64 counter RNG and the group decoder.
//
// Layout in HBM:
//   genes     uint8  [item][stage][Jpad]      stage-major rows, Jpad = round_up(J, 16)
//   procT     fp64   [stage_off[s]+m][J+1]    one column per (stage, machine); slot J = 0 pad
//   release / due fp64 [J];  rel_order u16 [J] (stage-0 dispatch order, model.cpp:98-105)
//   pseudo members u64 [member][W]           bit i of the reference BitChromosome at
//                                            word i/64, bit i%64 (pseudo.cpp:22-27 mask order)
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

namespace ffsga_dev {

constexpr uint64_t kGamma = 0x9E3779B97F4A7C15ULL;
constexpr int kMaxMachines = 32;  // lanes per decoder group: one lane per machine of a stage

struct DevInst {
    int J, S, Jpad, maxM;
    int bits_per_job, total_bits, words;
    int cta_sync;   // decoder stage barriers: 1 = CTA-wide (shared procT slice in L1), 0 = per warp
    int max_warps;  // decoder CTA size cap (0 = smem-limited, at most 16)
    int algo;       // decoder: 0 = k-way merge of per-source lists, 1 = per-stage bucket sort
    int bshift;     // bucket decoder: J << bshift histogram buckets per stage
    int check_selftest;  // checked build: K1 reports a deliberate failure (proves the channel)
    int pk_bits;    // K1 fast pass with packed heads: low pk_bits of a ready time's bits hold the
                    // job id (0 = off; needs every ready time >= +0.0, see capi.cu)
    double weight, emax;
    const int* M;               // [S]
    const int* stage_off;       // [S+1]
    const int* bps;             // bits per stage [S]
    const int* sbo;             // stage bit offset inside one job [S+1]
    const double* procT;        // [(stage_off[s]+m)*(J+1) + j]
    const double* release;      // [J]
    const double* due;          // [J]
    const uint16_t* rel_order;  // [J]
};

// ---------------------------------------------------------------- SplitMix64 (rng.hpp:14-62)
// Output k (0-based) of Rng(seed) is mix(seed + (k+1)*gamma): the stream is counter-based,
// so any lane can jump to any draw.
__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}
__device__ __forceinline__ uint64_t draw(uint64_t seed, uint64_t k) {
    return mix64(seed + (k + 1ULL) * kGamma);
}
// derive_seed(base, key) = output `key` of Rng(base)   (rng.hpp:55-58)
__device__ __forceinline__ uint64_t derive_seed(uint64_t base, uint64_t key) { return draw(base, key); }
// next_unit (rng.hpp:26-28): exact 53-bit integer times 2^-53
__device__ __forceinline__ double unit_of(uint64_t u) {
    return __dmul_rn(__ull2double_rn(u >> 11), 0x1.0p-53);
}
// next_index (rng.hpp:39-43): truncation of an RNE fp64 product, clamped
__device__ __forceinline__ int index_of(uint64_t u, int n) {
    int v = __double2int_rz(__dmul_rn(unit_of(u), static_cast<double>(n)));
    return v < n ? v : n - 1;
}
// next_coin (rng.hpp:45): unit < p  <=>  (u >> 11) < ceil(p * 2^53)  (thr precomputed on host)
__device__ __forceinline__ bool coin_of(uint64_t u, uint64_t thr) { return (u >> 11) < thr; }

// ---------------------------------------------------------------- group decoder (K1)
// One group of G lanes decodes one chromosome; lane m owns machine m of the current stage.
// Shared-memory block per group (bytes):
struct GroupLayout {
    int off_next, off_tail, off_row, bytes;
};
__host__ __device__ inline int align16(int x) { return (x + 15) & ~15; }
__host__ __device__ inline GroupLayout group_layout(int J, int Jpad, int G) {
    GroupLayout g;
    int ready = align16(8 * (J + 1 + G * G));         // fp64 node values (jobs, END, dummies)
    int next = align16(2 * (J + 1 + G * G));          // u16 links + G*G list dummies
    int tail = align16(2 * G * G);                    // u16 tail[m][dst]
    g.off_next = ready;
    g.off_tail = ready + next;
    g.off_row = ready + next + tail;
    g.bytes = g.off_row + Jpad;                       // u8 gene row of the next stage
    return g;
}

struct BucketLayout {
    int off_row, off_cnt, off_scat, off_fin, bytes, nb_cap, nbj;
};
// per group: keys fp64[J] | gene row u8[Jpad] | histogram u16[nb_cap] | scatter u16[J] | order u16[J]
// nbj = histogram buckets per stage (J << bshift, or J >> -bshift), split evenly over the machines
__host__ __device__ inline BucketLayout bucket_layout(int J, int Jpad, int G, int bshift) {
    BucketLayout b;
    b.nbj = bshift >= 0 ? (J << bshift) : (J >> -bshift);
    if (b.nbj < 1) b.nbj = 1;
    const int vec = 8 * G;  // u16 counters per lane-round of the vectorised scan
    b.nb_cap = ((b.nbj + 32 + vec - 1) / vec) * vec;
    b.off_row = align16(8 * J);
    b.off_cnt = b.off_row + align16(Jpad);
    b.off_scat = b.off_cnt + 2 * b.nb_cap;
    b.off_fin = b.off_scat + align16(2 * J);
    b.bytes = b.off_fin + align16(2 * J);
    return b;
}

struct BadTrack {  // first out-of-range gene in the next stage's dispatch order: min (ready, job)
    double c;
    int j;
    __device__ void reset() { c = __longlong_as_double(0x7FF0000000000000LL); j = 0x7FFFFFFF; }
    __device__ void consider(double cc, int jj) {
        if (cc < c || (cc == c && jj < j)) { c = cc; j = jj; }
    }
};

}  // namespace ffsga_dev
