// kernels.cu -- sm_100a kernels of the FFS hot path.
//
//   K1  k_eval            decode + evaluate a batch (Evaluator::score, model.cpp:61-120,183-195)
//   K2  k_random_rows     random assignment chromosomes (chromosome.cpp:68-74)
//   K3  k_cell_breed      cellular selection / two-point crossover / mutation (cellular.cpp:108-150)
//   K4  k_pseudo_breed    complementary-pair mask crossover (pseudo.cpp:11-29,59-82)
//   K6  k_commit          replacement, archive, best index, trace (cellular.cpp:164-189,
//                         pseudo.cpp:83-96, solver.cpp:111-123)
//   K5  migration         sort_island order + install with representation change (migration.cpp:47-69)
//   K7  k_eval<SCHED>     full timetable of one chromosome (model.cpp:124-139)
//
// All fp64 arithmetic uses explicit round-to-nearest intrinsics (no FMA contraction) so results
// are bit-identical to the reference built with -ffp-contract=off (proj/src/CMakeLists.txt:16).
#include <cub/cub.cuh>
#include <cuda_pipeline.h>

#include <algorithm>
#include <cstdlib>
#include <type_traits>

#include "launch.h"
#include "decoder_common.cuh"

namespace ffsga_dev {

namespace {

// ---------------------------------------------------------------------------- K1 decoder
// Design: one group of G lanes per chromosome, lane m owns machine m of the
// current stage; every group of a CTA advances stage by stage in lockstep (__syncthreads at
// stage boundaries) so the CTA shares one stage slice of the processing-time table in L1.
//
// Per-group shared memory (node = job 0..J-1, END = J, list dummies J+1+src*G+dst):
//   link[node] u16  -- next job of the node's list
//   lval[node] fp64 -- ready time (previous-stage completion) of link[node]; +inf after END
//   tail[G*G]  u16  -- tail node of each outgoing list of this stage
//   two gene rows   -- stage s+1 (routing of this stage) and s+2 (cp.async prefetch)
// Carrying the successor's ready time in the node lets a pop fetch both the next head and its
// key with two independent loads.  After the last stage lval[j] holds job j's completion.

// One stage of the list schedule for the group's chromosome (model.cpp:68-95).
// Lane m (< Ms) merges the NS incoming per-source lists of jobs routed to machine m (each list
// is sorted by completion because completions on one machine strictly increase), which
// reproduces the (ready, job) sort of model.cpp:72-75 restricted to machine m, then runs the
// machine's fp64 recurrence start = max(ready, avail), completion = start + p (84-87) and
// appends the job to its outgoing list (m -> gene of the next stage).  Branch-free body:
// out-of-range next-stage genes land in lists nobody reads and are reported after the stage.
// PK: packed heads (decoder_common.cuh pk_*): node values are keys, the link region holds the
// dropped low bits of each job's ready time (indexed by job), and the popped job comes out of
// head 0's key; ready-only pass only (not EXACT, not SCHED).
template <int G, int NS, bool SCHED, bool LAST, bool EARLY, bool EXACT, int DEPTH, bool PK>
__device__ __forceinline__ void stage_pass(const DevInst& I, int s, int Mprev, int Ms, int Mnext,
                                           int m, bool work, double* __restrict__ lval,
                                           uint16_t* __restrict__ link, uint16_t* __restrict__ tail,
                                           const uint8_t* __restrict__ row, const EvalItems& W, bool& tie) {
    const int J = I.J;
    const int END = J;
    constexpr bool last = LAST;
    const double* pcol = I.procT + (size_t)(I.stage_off[s] + (m < Ms ? m : 0)) * (J + 1);
    // The column pointer and the gene row's shared-window address are pinned in registers:
    // left to itself the compiler refolds them into the pop loop (a 64-bit index add + shift +
    // constant-bank reload of procT per pop, and S2R SR_CgaCtaId + LEA per pop for the row).
    asm volatile("" : "+l"(pcol));
    unsigned row_s = (unsigned)__cvta_generic_to_shared(row);
    asm volatile("" : "+r"(row_s));
    static_assert(!PK || (!EXACT && !SCHED), "packed heads serve the ready-only pass");
    const unsigned mask = PK ? (1u << I.pk_bits) - 1u : 0u;
    double hv[NS];
    int hj[NS];
#pragma unroll
    for (int k = 0; k < NS; ++k) {
        const bool live = work && m < Ms && k < Mprev;
        const int node = J + 1 + k * G + m;
        if (PK) {
            hv[k] = live ? lval[node] : pk_sentinel(END, mask);
            FFSGA_CHECK(pk_job(hv[k], mask) <= END, 1, pk_job(hv[k], mask), s);
        } else {
            hj[k] = live ? (int)link[node] : END;
            hv[k] = live ? lval[node] : dinf();
            FFSGA_CHECK(hj[k] <= END, 1, hj[k], s);
        }
    }
    if (PK)
        heads_sort_pk<NS>(hv);
    else
        heads_sort<NS>(hv, hj);
    // the job at head 0
    auto head = [&]() -> int {
        if (PK) return pk_job(hv[0], mask);
        return hj[0];
    };
    uint16_t* mytail = tail + m * G;
    if (!last) {
#pragma unroll
        for (int d = 0; d < G; ++d) mytail[d] = (uint16_t)(J + 1 + m * G + d);
    }
#ifdef FFSGA_CHECKED
    unsigned long long ck_n = 0, ck_s1 = 0, ck_s2 = 0;
#endif
    stage_barrier(I.cta_sync);
    if (work && m < Ms) {
        // Software pipelined by two pops: pop i is retired (recurrence, list append, stores) in
        // iteration i+2, so its processing-time load (an L1 miss whenever the stage slice does
        // not fit L1, i.e. an L2 round trip) has two head insertions to arrive.  The loop is
        // unrolled twice with one pending slot per half (A, B): each half retires the slot it
        // is about to refill -- the oldest pending pop -- and then loads straight into it, so
        // no register copy waits on a load (a copy at the loop end did: a third of all K1 stall
        // samples once sat on one IMAD.MOV behind the procT load).  DEPTH 3: three slots, three
        // pops in flight.  The successor link/value of the popped job is loaded before the
        // retire (EARLY; the other order measured 139.0 vs 149.0 C3 generations/s); the
        // retire's stores cannot alias it: the popped job has not been dispatched at this stage,
        // so it is neither a tail nor a dummy of the stage's outgoing lists.
        double avail = 0.0;
        struct Pend {
            double br, p;  // ready time, processing time
            int g, j;      // next-stage gene, job (END: empty)
        };
        // ready times of the two pending pops; NaN (equal to nothing) until a slot is filled
        const double qnan = __longlong_as_double(0x7FF8000000000000LL);
        Pend A{qnan, 0.0, 0, END}, B{qnan, 0.0, 0, END};
        bool eq = false;  // two consecutive pops with equal ready times (ready-only order)
        // PK: minimum over pops of the bits in which a pop's key differs from the previous pop's
        // ready time above the job bits; 0 = the two agree there (possibly out of order)
        unsigned tacc = 0xFFFFFFFFu;
        auto retire = [&](const Pend& q) {
            const double start = (q.br < avail) ? avail : q.br;  // std::max(ready, avail)
            const double c = __dadd_rn(start, q.p);
            avail = c;
            if (SCHED) {
                const int at = q.j * I.S + s;
                W.smachine[at] = m;
                W.sstart[at] = start;
                W.scomp[at] = c;
            }
            if (!last) {
                const int d = min(q.g, G - 1);
                const int t = mytail[d];
                FFSGA_CHECK(t != END && t < J + 1 + G * G, 4, t, q.j);
                if (PK) {
                    lval[t] = pk_pack(c, q.j, mask);
                    link[q.j] = (uint16_t)pk_low(c, mask);  // q.j's next ready time, low bits
                } else {
                    link[t] = (uint16_t)q.j;
                    lval[t] = c;
                }
                mytail[d] = (uint16_t)q.j;
            } else {
                lval[q.j] = c;  // final completion (the node was consumed by its pop)
            }
        };
        // one pop into slot q (which holds the oldest pending pop, retired first)
#ifdef FFSGA_CHECKED
        // invariants of the merge: every pop is a job, its successor a node, the popped ready
        // times are sorted (strictly in (ready, job) order for the exact comparator), and over
        // the group's lanes the stage pops every job exactly once (count and two checksums)
        double ck_v = -dinf();
        int ck_j = -1;
#endif
        auto pop = [&](Pend& q, const Pend& prev, int bj) {
            if (PK)  // keys agreeing above the job bits: possibly out of (ready, job) order
                tacc = min(tacc, pk_high_diff(hv[0], prev.br, mask));
            else if (!EXACT)
                eq |= hv[0] == prev.br;  // the pops are sorted by ready time: ties adjoin
#ifdef FFSGA_CHECKED
            FFSGA_CHECK(bj >= 0 && bj < J, 2, bj, s);
            if (EXACT) {
                FFSGA_CHECK(key_lt(ck_v, ck_j, hv[0], bj), 6, bj, s);
                ck_v = hv[0];
            } else if (PK) {  // packed: sorted above the job bits (below them a flagged tie)
                const double hi_part = pk_value(hv[0], 0u, mask);
                FFSGA_CHECK(!(hi_part < ck_v), 5, bj, s);
                ck_v = hi_part;
            } else {
                FFSGA_CHECK(!(hv[0] < ck_v), 5, bj, s);
                ck_v = hv[0];
            }
            ck_j = bj;
            ck_n += 1;
            ck_s1 += (unsigned long long)bj;
            ck_s2 += (unsigned long long)bj * (unsigned long long)bj;
#endif
            int nh;
            double nr;
            if (PK) {  // the successor's key; bj's own ready time, low bits
                nr = lval[bj];
                nh = link[bj];
            } else if (EARLY) {
                nh = link[bj];
                nr = lval[bj];
            }
            FFSGA_CHECK(PK || !EARLY || nh <= END, 3, nh, bj);
            FFSGA_CHECK(!PK || pk_job(nr, mask) <= END, 3, pk_job(nr, mask), bj);
            if (q.j != END) retire(q);
            q.br = PK ? pk_value(hv[0], (unsigned)nh, mask) : hv[0];
            q.p = __ldg(pcol + (unsigned)bj);  // unsigned index: one IMAD.WIDE.U32
            if (last) {
                q.g = 0;
            } else {
                unsigned g;
                asm volatile("ld.shared.u8 %0, [%1];" : "=r"(g) : "r"(row_s + (unsigned)bj));
                q.g = (int)g;
            }
            q.j = bj;
            if (!PK && !EARLY) {
                nh = link[bj];
                nr = lval[bj];
            }
            if (PK)
                heads_replace_min_pk<NS>(hv, nr);
            else
                heads_replace_min<NS, EXACT>(hv, hj, nr, nh);
        };
        if constexpr (DEPTH == 2 || DEPTH == 4) {
            bool a_older = true;  // which pending slot holds the older pop at loop exit
            if constexpr (DEPTH == 4) {
            // "DEPTH 4": the two-slot pipeline unrolled four pops deep (J >= 300): the register
            // copies the compiler inserts at the loop's back edge are paid once per four pops,
            // and the longer body schedules better (500x20 +2.4 %; at 100x10 the larger body
            // costs 11 %, so small instances keep the two-pop body)
            while (true) {
                int bj = head();
                if (bj == END) break;
                pop(A, B, bj);
                bj = head();
                if (bj == END) {
                    a_older = false;
                    break;
                }
                pop(B, A, bj);
                bj = head();
                if (bj == END) break;
                pop(A, B, bj);
                bj = head();
                if (bj == END) {
                    a_older = false;
                    break;
                }
                pop(B, A, bj);
            }
            } else {
            while (true) {
                int bj = head();
                if (bj == END) break;
                pop(A, B, bj);
                bj = head();
                if (bj == END) {
                    a_older = false;
                    break;
                }
                pop(B, A, bj);
            }
            }
            tie |= eq | (tacc == 0u);
            if (a_older) {
                if (A.j != END) retire(A);
                if (B.j != END) retire(B);
            } else {
                if (B.j != END) retire(B);
                if (A.j != END) retire(A);
            }
        } else {  // three pops in flight (large J: the procT slice misses L1 more often)
            Pend C{qnan, 0.0, 0, END};
            int exit_at = 0;  // the slot the loop stopped before holds the oldest pending pop
            while (true) {  // unrolled six pops deep (see DEPTH 4)
                int bj = head();
                if (bj == END) break;
                pop(A, C, bj);
                bj = head();
                if (bj == END) {
                    exit_at = 1;
                    break;
                }
                pop(B, A, bj);
                bj = head();
                if (bj == END) {
                    exit_at = 2;
                    break;
                }
                pop(C, B, bj);
                bj = head();
                if (bj == END) break;
                pop(A, C, bj);
                bj = head();
                if (bj == END) {
                    exit_at = 1;
                    break;
                }
                pop(B, A, bj);
                bj = head();
                if (bj == END) {
                    exit_at = 2;
                    break;
                }
                pop(C, B, bj);
            }
            tie |= eq | (tacc == 0u);
            if (exit_at == 0) {
                if (A.j != END) retire(A);
                if (B.j != END) retire(B);
                if (C.j != END) retire(C);
            } else if (exit_at == 1) {
                if (B.j != END) retire(B);
                if (C.j != END) retire(C);
                if (A.j != END) retire(A);
            } else {
                if (C.j != END) retire(C);
                if (A.j != END) retire(A);
                if (B.j != END) retire(B);
            }
        }
        if (!last) {
#pragma unroll
            for (int d = 0; d < G; ++d) {
                const int t = mytail[d];
                if (PK) {
                    lval[t] = pk_sentinel(END, mask);
                } else {
                    link[t] = (uint16_t)END;
                    lval[t] = dinf();
                }
            }
        }
    }
#ifdef FFSGA_CHECKED
#pragma unroll
    for (int off = G / 2; off > 0; off >>= 1) {
        ck_n += __shfl_xor_sync(kFull, ck_n, off, G);
        ck_s1 += __shfl_xor_sync(kFull, ck_s1, off, G);
        ck_s2 += __shfl_xor_sync(kFull, ck_s2, off, G);
    }
    if (work && m == 0) {
        const unsigned long long Ju = (unsigned long long)J;
        FFSGA_CHECK(ck_n == Ju, 7, ck_n, s);
        FFSGA_CHECK(ck_s1 == Ju * (Ju - 1) / 2, 8, ck_s1, s);
        FFSGA_CHECK(ck_s2 == (Ju - 1) * Ju * (2 * Ju - 1) / 6, 9, ck_s2, s);
    }
#endif
    stage_barrier(I.cta_sync);
}

template <int G, bool SCHED, bool EARLY, bool EXACT, int DEPTH, bool PK>
__device__ __forceinline__ void dispatch_stage(const DevInst& I, int s, int Mprev, int Ms, int Mnext,
                                               int m, bool work, double* lval, uint16_t* link,
                                               uint16_t* tail, const uint8_t* row, const EvalItems& W,
                                               bool& tie) {
#define FFSGA_STAGE(NS_)                                                                           \
    if constexpr (NS_ <= G) {                                                                       \
        if (Mprev <= NS_) {                                                                         \
            if (Mnext)                                                                              \
                stage_pass<G, NS_, SCHED, false, EARLY, EXACT, DEPTH, PK>(I, s, Mprev, Ms, Mnext, m, work, lval, link, tail, \
                                                               row, W, tie);                        \
            else                                                                                    \
                stage_pass<G, NS_, SCHED, true, EARLY, EXACT, DEPTH, PK>(I, s, Mprev, Ms, Mnext, m, work, lval, link, tail, \
                                                              row, W, tie);                         \
            return;                                                                                 \
        }                                                                                           \
    }
    FFSGA_STAGE(1)
    FFSGA_STAGE(2)
    FFSGA_STAGE(3)
    FFSGA_STAGE(4)
    FFSGA_STAGE(5)
    FFSGA_STAGE(6)
    FFSGA_STAGE(7)
    FFSGA_STAGE(8)
    FFSGA_STAGE(16)
    FFSGA_STAGE(32)
#undef FFSGA_STAGE
}

// Out-of-range genes of stage s+1 (rare): walk lane m's outgoing lists (their nodes carry each
// job's stage-s completion) and return the first offender in stage s+1 dispatch order, i.e.
// the minimum (completion, job) among jobs whose next-stage gene is >= Mnext.
template <int G, bool PK>
__device__ __forceinline__ void find_bad(const DevInst& I, int m, int Ms, int Mnext, const double* lval,
                                         const uint16_t* link, const uint8_t* row, BadTrack& bad) {
    const int J = I.J;
    const unsigned mask = PK ? (1u << I.pk_bits) - 1u : 0u;
    if (m >= Ms) return;
    for (int d = 0; d < G; ++d) {
        int node = J + 1 + m * G + d;
        while (true) {
            const int j = PK ? pk_job(lval[node], mask) : (int)link[node];
            if (j == J) break;
            if (row[j] >= Mnext) bad.consider(PK ? pk_value(lval[node], link[j], mask) : lval[node], j);
            node = j;
        }
    }
}

// (512, 1): without the explicit minimum ptxas may cap the small-body variants at 64 registers
// (with spills) to fit two 512-thread CTAs, which the shared-memory budget never allows anyway
template <int G, bool SCHED, int DEPTH, bool PK>
__global__ void __launch_bounds__(512, 1) k_eval(DevInst I, EvalItems W, int groups_per_cta, GroupLayout GL) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int gw = lane / G;
    const int m = lane % G;
    const int gid = threadIdx.x / G;
    unsigned char* gb = smem + (size_t)gid * GL.bytes;
    double* lval = reinterpret_cast<double*>(gb);
    uint16_t* link = reinterpret_cast<uint16_t*>(gb + GL.off_next);
    uint16_t* tail = reinterpret_cast<uint16_t*>(gb + GL.off_tail);
    uint8_t* const row_a = gb + GL.off_row;
    const int J = I.J, S = I.S;
    const int END = J;
    const long long n = W.n_dev ? *W.n_dev + W.n : W.n;  // fused GA list: n cells + device count
    FFSGA_CHECK(!I.check_selftest, 99, blockIdx.x, threadIdx.x);

    // All groups of the CTA share the item loop (CTA-uniform bounds: stage barriers).  A launch
    // that owns the GPU deals items round-robin over the CTAs (group g of CTA b takes item
    // base + g * grid + b), so a final partial round spreads over every SM: a round lasts one
    // chromosome's decode however many groups it holds, and thinly filled SMs decode faster.
    // Launches sharing the GPU (joint GA step) take contiguous blocks instead, so CTAs without
    // items in the last round exit and hand their SM to the other launch.
    const long long stride = (long long)gridDim.x * groups_per_cta;
    for (long long base = W.deal ? 0 : (long long)blockIdx.x * groups_per_cta; base < n; base += stride) {
        const long long item = W.deal ? base + (long long)gid * gridDim.x + blockIdx.x : base + gid;
        const bool active = item < n;
        const uint8_t* genes = active ? (W.ptrs ? W.ptrs[item] : W.base + item * W.stride) : nullptr;

        // One decode of the group's chromosome (stage-0 routing, then every stage).  `work`
        // enters as "decode this group" and leaves false when a gene is out of range; `tie`
        // reports equal consecutive ready times under the ready-only pop order.
        auto decode = [&](auto exact_tag, bool& work, bool& tie, unsigned long long& errc) {
            constexpr bool EXACT = decltype(exact_tag)::value;
            constexpr bool PKD = PK && !EXACT;  // packed heads in the ready-only pass
            const unsigned mask = PKD ? (1u << I.pk_bits) - 1u : 0u;
            if (work) prefetch_row<G>(I, genes, 0, m, row_a);
            tail[m] = (uint16_t)(J + 1 + m);  // virtual source 0 -> machine m of stage 0
            __pipeline_wait_prior(0);
            __syncwarp();

            // ---- stage-0 routing: release order (model.cpp:98-105) split per machine, in order;
            // node values are release times.  G consecutive jobs are linked per match_any.
            const int M0 = I.M[0];
            int bad_k = 0x7FFFFFFF;
            for (int b0 = 0; b0 < J; b0 += G) {
                const int k = b0 + m;
                const bool valid = work && k < J;
                const int j = valid ? (int)I.rel_order[k] : 0;
                const int d = valid ? (int)row_a[j] : 0;
                const bool good = valid && d < M0;
                if (valid && !good) bad_k = min(bad_k, k);
                const double rel = valid ? __ldg(I.release + j) : 0.0;
                const unsigned key = good ? (((unsigned)gw << 8) | (unsigned)d) : (0x10000u | (unsigned)lane);
                const unsigned peers = __match_any_sync(kFull, key);
                const unsigned below = peers & ((1u << lane) - 1u);
                const unsigned above = peers & ~((2u << lane) - 1u);
                const int pred_lane = below ? (31 - __clz(below)) : lane;
                const int pred_j = __shfl_sync(kFull, j, pred_lane);
                int t = 0;
                if (good && !below) t = tail[d];
                __syncwarp();
                if (good) {
                    const int node = below ? pred_j : t;
                    if (PKD) {
                        lval[node] = pk_pack(rel, j, mask);
                        link[j] = (uint16_t)pk_low(rel, mask);
                    } else {
                        link[node] = (uint16_t)j;
                        lval[node] = rel;
                    }
                }
                if (good && !above) tail[d] = (uint16_t)j;
                __syncwarp();
            }
            if (work) {
                const int t = tail[m];
                FFSGA_CHECK(t != END && t < J + 1 + G * G, 10, t, m);
                if (PKD) {
                    lval[t] = pk_sentinel(END, mask);
                } else {
                    link[t] = (uint16_t)END;
                    lval[t] = dinf();
                }
            }
            bad_k = group_min_int<G>(bad_k);
            if (work && bad_k != 0x7FFFFFFF) {
                work = false;
                errc = ((unsigned long long)item << 32) | (unsigned long long)I.rel_order[bad_k];
            }

            // ---- stages
            int Mprev = 1;
            for (int s = 0; s < S; ++s) {
                const int Ms = I.M[s];
                const int Mnext = (s + 1 < S) ? I.M[s + 1] : 0;
                const uint8_t* row = row_a;
                __syncwarp();  // every lane is done with row s
                if (work && s + 1 < S) prefetch_row<G>(I, genes, s + 1, m, row_a);
                if (work && s + 2 < S)  // warm L2 with row s+2 (no shared memory spent on it)
                    for (int v = m; v * 128 < I.Jpad; v += G)
                        asm volatile("prefetch.global.L2 [%0];" ::"l"(genes + (size_t)(s + 2) * I.Jpad + v * 128));
                __pipeline_wait_prior(0);  // row s+1 has landed
                __syncwarp();
                bool row_bad = false;
                if (Mnext) row_bad = row_has_bad<G>(I, row, m, Mnext, work);
                dispatch_stage<G, SCHED, true, EXACT, DEPTH, PKD>(I, s, Mprev, Ms, Mnext, m, work, lval, link, tail, row,
                                                             W, tie);
                if (__any_sync(kFull, row_bad)) {
                    // first offending job in stage s+1 dispatch order: min (ready, job) among them
                    BadTrack bad;
                    bad.reset();
                    if (row_bad && work) find_bad<G, PKD>(I, m, Ms, Mnext, lval, link, row, bad);
                    double bc = bad.c;
                    int bj = bad.j;
                    group_min_key<G>(bc, bj);
                    if (row_bad && work && bj != 0x7FFFFFFF) {
                        work = false;
                        errc = ((unsigned long long)item << 32) | ((unsigned long long)(s + 1) << 16) |
                               (unsigned long long)bj;
                    }
                }
                Mprev = Ms;
            }
            __pipeline_wait_prior(0);
        };

        bool work = active, tie = false;
        unsigned long long errc = kNoErr;  // first out-of-range gene, reported once the order is exact
        decode(std::false_type{}, work, tie, errc);
        // Equal ready times met under the ready-only order (integer-valued instances; never seen
        // with continuous processing times): decode those chromosomes again in (ready, job)
        // order.  CTA-uniform decision, because the stage passes contain CTA barriers.  A group
        // that also met an out-of-range gene after the tie is redone too: which job the reference
        // names first depends on the exact completions (model.cpp:81-83), so the error of the
        // exact pass replaces that of the fast one.
        const bool any_tie = I.cta_sync ? (__syncthreads_or(tie) != 0) : __any_sync(kFull, tie);
        if (any_tie) {
            unsigned gt = tie ? 1u : 0u;
#pragma unroll
            for (int off = G / 2; off > 0; off >>= 1) gt |= __shfl_xor_sync(kFull, gt, off, G);
            bool redo = gt != 0 && active, tie2 = false;
            unsigned long long errc2 = kNoErr;
            decode(std::true_type{}, redo, tie2, errc2);
            if (gt) {
                work = redo;
                errc = errc2;
            }
        }
        if (errc != kNoErr && m == 0 && W.err) atomicMin(W.err, errc);

        // ---- report_from_completions (model.cpp:107-120); completions are in lval[0..J)
        double mk = 0.0;
        if (work) {
            for (int j = m; j < J; j += G) {
                const double c = lval[j];
                mk = (mk < c) ? c : mk;
                const double t = __dsub_rn(c, __ldg(I.due + j));
                lval[j] = (0.0 < t) ? t : 0.0;  // std::max(0.0, c - due)
            }
        }
        mk = group_max<G>(mk);
        __syncwarp();
        if (work && m == 0) {
            double T = 0.0;  // sequential in job order: the fp64 sum is order dependent
            for (int j = 0; j < J; ++j) T = __dadd_rn(T, lval[j]);
            const double obj = __dadd_rn(__dmul_rn(I.weight, T), mk);
            const double f = __dsub_rn(I.emax, obj);
            W.obj[item] = obj;
            W.fit[item] = (f < 0.0) ? 0.0 : f;  // std::max(emax - obj, 0.0)
            if (W.mk) W.mk[item] = mk;
            if (W.td) W.td[item] = T;
        }
        stage_barrier(I.cta_sync);
    }
}


// ---------------------------------------------------------------------------- K1b bucket decoder
// Alternative K1 (FFSGA_EVAL_ALGO=bucket): the per-stage (ready, job) order of model.cpp:72-75,
// restricted to each machine, is built by a counting sort instead of a k-way merge, so only the
// machine recurrence stays serial.  Per stage, all G lanes of the group work on all J jobs:
//   P1  bucket = (machine, floor((ready - lo) * NBd / (hi - lo))) -> u16 histogram (smem atomics);
//       the map ready -> bucket is monotone (RN sub/mul and truncation never invert an order),
//       so buckets are ordered like their keys and only jobs inside one bucket need comparing;
//   P2  exclusive scan of the histogram (bucket start offsets);
//   P3  scatter jobs to their bucket (atomic cursor; order inside a bucket arbitrary);
//   P4  exact rank inside the bucket by (ready, job) -> final per-machine dispatch order;
//   P5  lane m runs machine m's recurrence start = max(ready, avail), C = start + p
//       (model.cpp:84-87) over its jobs in order, writing C in place of ready.
// Stage 0 sorts by the release rank (distinct integers; model.cpp:98-105) and reads the release
// times in P5.  lo/hi of the next stage are the first/last completion of each machine (non-
// decreasing because processing times are >= 0).  Ties of equal ready times land in one bucket
// and are ordered by job in P4, so no assumption on distinct completions is needed.
template <int G>
__device__ __forceinline__ int group_excl_scan(int v, int m, int& total) {
    int x = v;
#pragma unroll
    for (int off = 1; off < G; off <<= 1) {
        const int y = __shfl_up_sync(kFull, x, off, G);
        if (m >= off) x += y;
    }
    total = __shfl_sync(kFull, x, G - 1, G);
    return x - v;
}

struct BucketMap {
    double lo, scale;
    int nbd;
    __device__ __forceinline__ int operator()(double key, int g) const {
        const unsigned b = __double2uint_rz(__dmul_rn(__dsub_rn(key, lo), scale));
        return g * nbd + (int)min(b, (unsigned)(nbd - 1));
    }
};

__device__ __forceinline__ unsigned cnt_add(uint16_t* cnt, int idx) {
    unsigned* w = reinterpret_cast<unsigned*>(cnt) + (idx >> 1);
    const int sh = (idx & 1) * 16;
    return (atomicAdd(w, 1u << sh) >> sh) & 0xFFFFu;
}

template <int G, bool SCHED>
__global__ void __launch_bounds__(512) k_eval_bkt(DevInst I, EvalItems W, int groups_per_cta, BucketLayout BL) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = threadIdx.x & 31;
    const int m = lane % G;
    const int gid = threadIdx.x / G;
    unsigned char* gb = smem + (size_t)gid * BL.bytes;
    double* keys = reinterpret_cast<double*>(gb);
    uint8_t* const row = gb + BL.off_row;
    uint16_t* cnt = reinterpret_cast<uint16_t*>(gb + BL.off_cnt);
    uint16_t* scat = reinterpret_cast<uint16_t*>(gb + BL.off_scat);
    uint16_t* fin = reinterpret_cast<uint16_t*>(gb + BL.off_fin);
    const int J = I.J, S = I.S;
    const long long n = W.n_dev ? *W.n_dev + W.n : W.n;  // fused GA list: n cells + device count

    for (long long base = (long long)blockIdx.x * groups_per_cta; base < n;
         base += (long long)gridDim.x * groups_per_cta) {
        const long long item = base + gid;
        const bool active = item < n;
        const uint8_t* genes = nullptr;
        if (active) {
            genes = W.ptrs ? W.ptrs[item] : W.base + item * W.stride;
            prefetch_row<G>(I, genes, 0, m, row);
            for (int k = m; k < J; k += G) keys[I.rel_order[k]] = (double)k;  // stage-0 key: release rank
        }
        bool work = active;
        double lo = 0.0, hi = (double)(J - 1);
        for (int s = 0; s < S; ++s) {
            const int Ms = I.M[s];
            const int nbd = (BL.nbj + Ms - 1) / Ms;
            const int nb = Ms * nbd;
            BucketMap bm;
            bm.lo = lo;
            bm.nbd = nbd;
            {
                const double span = __dsub_rn(hi, lo);
                // any positive scale keeps the map monotone; fp32 reciprocal (no fp64 divide)
                bm.scale = (span > 0.0) ? (double)__fmul_rn((float)nbd, __frcp_rn((float)span)) : 0.0;
            }
            // clear the histogram (16 B stores)
            uint4* c4 = reinterpret_cast<uint4*>(cnt);
            const int nvec = (nb + 7) >> 3;
            for (int v = m; v < nvec; v += G) c4[v] = make_uint4(0, 0, 0, 0);
            __pipeline_wait_prior(0);  // gene row s has landed
            __syncwarp();

            // P1: histogram; out-of-range genes tracked as (key, job) = dispatch order
            BadTrack bad;
            bad.reset();
            bool any_bad = false;
            if (work) {
#pragma unroll 4
                for (int j = m; j < J; j += G) {
                    const double k = keys[j];
                    const int g = row[j];
                    if (g < Ms) {
                        const int idx = bm(k, g);
                        atomicAdd(reinterpret_cast<unsigned*>(cnt) + (idx >> 1), 1u << ((idx & 1) * 16));
                    } else {
                        any_bad = true;
                        bad.consider(k, j);
                    }
                }
            }
            if (__any_sync(kFull, any_bad)) {
                double bc = bad.c;
                int bj = bad.j;
                group_min_key<G>(bc, bj);
                if (work && bj != 0x7FFFFFFF) {
                    work = false;
                    if (m == 0 && W.err)
                        atomicMin(W.err, ((unsigned long long)item << 32) | ((unsigned long long)s << 16) |
                                             (unsigned long long)bj);
                }
            }
            __syncwarp();

            // P2: exclusive scan of the u16 histogram; lane m owns a contiguous run of vectors
            {
                const int per = (nvec + G - 1) / G;
                const int v0 = m * per, v1 = min(v0 + per, nvec);
                int sum = 0;
                for (int v = v0; v < v1; ++v) {
                    const uint4 x = c4[v];
                    sum += (int)((x.x & 0xFFFF) + (x.x >> 16) + (x.y & 0xFFFF) + (x.y >> 16) + (x.z & 0xFFFF) +
                                 (x.z >> 16) + (x.w & 0xFFFF) + (x.w >> 16));
                }
                int total;
                unsigned run = (unsigned)group_excl_scan<G>(sum, m, total);
                auto excl = [&run](unsigned w) {
                    const unsigned a = w & 0xFFFF, b = w >> 16;
                    const unsigned o = run | ((run + a) << 16);
                    run += a + b;
                    return o;
                };
                for (int v = v0; v < v1; ++v) {
                    uint4 x = c4[v];
                    x.x = excl(x.x);
                    x.y = excl(x.y);
                    x.z = excl(x.z);
                    x.w = excl(x.w);
                    c4[v] = x;
                }
            }
            __syncwarp();

            // P3: scatter to bucket slots
            if (work) {
#pragma unroll 4
                for (int j = m; j < J; j += G) {
                    const int idx = bm(keys[j], row[j]);
                    scat[cnt_add(cnt, idx)] = (uint16_t)j;
                }
            }
            __syncwarp();

            // P4: exact order inside each bucket; cnt[idx] now holds the end of bucket idx.  Buckets
            // hold ~2 jobs on average (uniform keys: Poisson), so the first kWin members are
            // compared branch-free and only larger buckets take the loop.
            if (work) {
                constexpr int kWin = 4;
#pragma unroll 2
                for (int p = m; p < J; p += G) {
                    const int j = scat[p];
                    const double k = keys[j];
                    const int idx = bm(k, row[j]);
                    const int st = idx ? (int)cnt[idx - 1] : 0;
                    const int en = cnt[idx];
                    int r = 0;
#pragma unroll
                    for (int u = 0; u < kWin; ++u) {
                        const int q = st + u;
                        const int jq = scat[q < en ? q : p];
                        r += (q < en && key_lt(keys[jq], jq, k, j)) ? 1 : 0;
                    }
                    for (int q = st + kWin; q < en; ++q) {
                        const int jq = scat[q];
                        r += key_lt(keys[jq], jq, k, j) ? 1 : 0;
                    }
                    fin[st + r] = (uint16_t)j;
                }
            }
            __syncwarp();
            // the row buffer is free: stage s+1's genes land during the recurrence
            if (work && s + 1 < S) prefetch_row<G>(I, genes, s + 1, m, row);
            if (work && s + 2 < S)
                for (int v = m; v * 128 < I.Jpad; v += G)
                    asm volatile("prefetch.global.L2 [%0];" ::"l"(genes + (size_t)(s + 2) * I.Jpad + v * 128));

            // P5: machine recurrence
            double first = dinf(), avail = -dinf();
            if (work && m < Ms) {
                const int b0 = m * nbd;
                const int begin = b0 ? (int)cnt[b0 - 1] : 0;
                const int finish = cnt[b0 + nbd - 1];
                const double* pcol = I.procT + (size_t)(I.stage_off[s] + m) * (J + 1);
                double av = 0.0;
                auto step = [&](int j, double r, double p) {
                    const double start = (r < av) ? av : r;  // std::max(ready, avail)
                    const double c = __dadd_rn(start, p);
                    av = c;
                    keys[j] = c;
                    if (SCHED) {
                        const int at = j * S + s;
                        W.smachine[at] = m;
                        W.sstart[at] = start;
                        W.scomp[at] = c;
                    }
                };
                // stage 0 reads release times (global), later stages the previous completions (smem)
                auto run = [&](auto rel_tag) {
                    constexpr bool REL = decltype(rel_tag)::value;
                    auto ready = [&](int j) { return REL ? __ldg(I.release + j) : keys[j]; };
                    int t = begin;
                    if (t < finish) {  // first job: its completion is the machine's minimum
                        const int j = fin[t];
                        step(j, ready(j), __ldg(pcol + (unsigned)j));
                        first = av;
                        ++t;
                    }
                    // four jobs per round: their loads are independent of the recurrence
                    for (; t + 3 < finish; t += 4) {
                        const int j0 = fin[t], j1 = fin[t + 1], j2 = fin[t + 2], j3 = fin[t + 3];
                        const double r0 = ready(j0), r1 = ready(j1), r2 = ready(j2), r3 = ready(j3);
                        const double p0 = __ldg(pcol + (unsigned)j0), p1 = __ldg(pcol + (unsigned)j1);
                        const double p2 = __ldg(pcol + (unsigned)j2), p3 = __ldg(pcol + (unsigned)j3);
                        step(j0, r0, p0);
                        step(j1, r1, p1);
                        step(j2, r2, p2);
                        step(j3, r3, p3);
                    }
                    for (; t < finish; ++t) {
                        const int j = fin[t];
                        step(j, ready(j), __ldg(pcol + (unsigned)j));
                    }
                };
                if (s == 0)
                    run(std::true_type{});
                else
                    run(std::false_type{});
                if (finish > begin) avail = av;
            }
            lo = group_min_d<G>(first);
            hi = group_max<G>(avail);
            stage_barrier(I.cta_sync);
        }
        __pipeline_wait_prior(0);

        // report_from_completions (model.cpp:107-120)
        double mk = 0.0;
        if (work) {
            for (int j = m; j < J; j += G) {
                const double c = keys[j];
                mk = (mk < c) ? c : mk;
                const double t = __dsub_rn(c, __ldg(I.due + j));
                keys[j] = (0.0 < t) ? t : 0.0;
            }
        }
        mk = group_max<G>(mk);
        __syncwarp();
        if (work && m == 0) {
            double T = 0.0;
            for (int j = 0; j < J; ++j) T = __dadd_rn(T, keys[j]);
            const double obj = __dadd_rn(__dmul_rn(I.weight, T), mk);
            const double f = __dsub_rn(I.emax, obj);
            W.obj[item] = obj;
            W.fit[item] = (f < 0.0) ? 0.0 : f;
            if (W.mk) W.mk[item] = mk;
            if (W.td) W.td[item] = T;
        }
        stage_barrier(I.cta_sync);
    }
}

// ---------------------------------------------------------------------------- K2 random rows
__global__ void __launch_bounds__(256) k_random_rows(DevInst I, uint8_t* out, long long stride, long long n,
                                                      unsigned long long base, long long first, int per_item) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const long long item = warp;
    const unsigned long long seed = per_item ? derive_seed(base, (unsigned long long)(first + item)) : base;
    const unsigned long long off = per_item ? 0ull : (unsigned long long)(first + item) * (unsigned long long)(I.J * I.S);
    uint8_t* dst = out + item * stride;
    const int words_per_row = I.Jpad / 4;
    for (int w = lane; w < I.S * words_per_row; w += 32) {
        const int s = w / words_per_row;
        const int j0 = (w % words_per_row) * 4;
        const int Ms = I.M[s];
        unsigned v = 0;
#pragma unroll
        for (int b = 0; b < 4; ++b) {
            const int j = j0 + b;
            if (j < I.J) {
                const unsigned g = (unsigned)index_of(draw(seed, off + (unsigned long long)(j * I.S + s)), Ms);
                v |= g << (8 * b);
            }
        }
        reinterpret_cast<unsigned*>(dst + (size_t)s * I.Jpad)[j0 / 4] = v;
    }
}

// int32 / uint8 job-major host layout -> device stage-major rows (255 marks out-of-range genes)
__global__ void __launch_bounds__(256) k_rows_from_int(DevInst I, const int32_t* gi, const uint8_t* gu,
                                                        uint8_t* rows, long long n) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const long long L = (long long)I.J * I.S;
    uint8_t* dst = rows + warp * (long long)I.S * I.Jpad;
    for (int idx = lane; idx < I.S * I.Jpad; idx += 32) {
        const int s = idx / I.Jpad, j = idx % I.Jpad;
        uint8_t v = 0;
        if (j < I.J) {
            if (gi) {
                const int32_t x = gi[warp * L + (long long)j * I.S + s];
                v = (x < 0 || x > 254) ? (uint8_t)255 : (uint8_t)x;
            } else {
                v = gu[warp * L + (long long)j * I.S + s];
            }
        }
        dst[idx] = v;
    }
}

__global__ void __launch_bounds__(256) k_rows_to_int(DevInst I, const uint8_t* rows, long long row_stride,
                                                      const long long* src_idx, int32_t* out, long long n) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const long long src = src_idx ? src_idx[warp] : warp;
    const uint8_t* r = rows + src * row_stride;
    const long long L = (long long)I.J * I.S;
    for (int g = lane; g < L; g += 32) {
        const int j = g / I.S, s = g % I.S;
        out[warp * L + g] = r[(size_t)s * I.Jpad + j];
    }
}

// ---------------------------------------------------------------------------- bit views
// int_to_bits (chromosome.cpp:28-42): gene (j,s) -> bits_per_stage[s] slot at j*bpj + sbo[s],
// MSB first.  bit_stage[r] = stage owning bit r of a job.  Packed LSB-first in u64 words.
__device__ __forceinline__ unsigned long long pack_word(const DevInst& I, const uint8_t* r, int w,
                                                         const uint16_t* bit_stage) {
    unsigned long long out = 0;
    const int b0 = w * 64;
    const int b1 = min(b0 + 64, I.total_bits);
    int job = b0 / I.bits_per_job;
    int rr = b0 - job * I.bits_per_job;
    for (int b = b0; b < b1; ++b) {
        const int s = bit_stage[rr];
        const int pos = rr - I.sbo[s];
        const int nb = I.bps[s];
        const unsigned v = r[(size_t)s * I.Jpad + job];
        out |= (unsigned long long)((v >> (nb - 1 - pos)) & 1u) << (b - b0);
        if (++rr == I.bits_per_job) { rr = 0; ++job; }
    }
    return out;
}

__global__ void __launch_bounds__(256) k_pack_bits(DevInst I, const uint8_t* rows, long long row_stride,
                                                    const long long* src_idx, unsigned long long* words,
                                                    const long long* dst_idx, long long n, int with_complement,
                                                    const uint16_t* bit_stage) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const long long src = src_idx ? src_idx[warp] : warp;
    const long long dst = dst_idx ? dst_idx[warp] : warp;
    const uint8_t* r = rows + src * row_stride;
    for (int w = lane; w < I.words; w += 32) {
        const unsigned long long x = pack_word(I, r, w, bit_stage);
        if (with_complement) {
            const int nb = min(64, I.total_bits - w * 64);
            const unsigned long long valid = nb == 64 ? ~0ull : ((1ull << nb) - 1ull);
            words[(2 * dst) * I.words + w] = x;
            words[(2 * dst + 1) * I.words + w] = (~x) & valid;  // complement (chromosome.cpp:61-66)
        } else {
            words[dst * I.words + w] = x;
        }
    }
}

// bits_to_int (chromosome.cpp:44-59): slot value MSB-first, modulo the stage's machines.
// bits_to_int (chromosome.cpp:44-59): slot value MSB-first, modulo the stage's machines.  The
// slot holds bps = max(1, bit_width(M-1)) bits, so value < 2^bps < 2M and the modulo is a single
// conditional subtraction.
__device__ __forceinline__ unsigned extract_gene(const unsigned long long* wv, int o, int nb, unsigned M) {
    const int w = o >> 6, sh = o & 63;
    unsigned long long x = wv[w] >> sh;
    if (sh + nb > 64) x |= wv[w + 1] << (64 - sh);
    const unsigned raw = (unsigned)(x & ((1ull << nb) - 1ull));  // bit o at position 0
    const unsigned val = __brev(raw) >> (32 - nb);               // bit o becomes the MSB
    return val >= M ? val - M : val;
}

// Four consecutive jobs per lane: a job's slots are contiguous, so when its bits fit 128
// (bits_per_job <= 128, e.g. 48 at 500x20x[2,8]) the lane loads the three words that can hold
// them once and cuts every gene out of a 128-bit register window; the four genes of a stage go
// out as one 32-bit store (the 32 lanes of a warp write 128 consecutive bytes of each stage row).
// Wider jobs read the words per gene.
__device__ __forceinline__ unsigned window_gene(unsigned long long lo, unsigned long long hi, int o, int nb,
                                                unsigned M) {
    const unsigned long long x = o >= 64 ? hi >> (o - 64) : (o ? (lo >> o) | (hi << (64 - o)) : lo);
    const unsigned raw = (unsigned)(x & ((1ull << nb) - 1ull));  // bit o at position 0
    const unsigned val = __brev(raw) >> (32 - nb);               // bit o becomes the MSB
    return val >= M ? val - M : val;
}

__device__ __forceinline__ void unpack_member(const DevInst& I, const unsigned long long* wv, uint8_t* dst,
                                              int lane) {
    if (I.bits_per_job > 128) {
        for (int j = lane; j < I.Jpad; j += 32) {
            const int base = j * I.bits_per_job;
            for (int s = 0; s < I.S; ++s)
                dst[(size_t)s * I.Jpad + j] =
                    j < I.J ? (uint8_t)extract_gene(wv, base + __ldg(I.sbo + s), __ldg(I.bps + s),
                                                    (unsigned)__ldg(I.M + s))
                            : (uint8_t)0;
        }
        return;
    }
    for (int q = lane; q < I.Jpad / 4; q += 32) {
        unsigned long long lo[4], hi[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int j = 4 * q + u;
            lo[u] = hi[u] = 0ull;
            if (j < I.J) {
                const int base = j * I.bits_per_job;
                const int w0 = base >> 6, sh = base & 63;
                const unsigned long long a = wv[w0];
                const unsigned long long b = w0 + 1 < I.words ? wv[w0 + 1] : 0ull;
                const unsigned long long c = w0 + 2 < I.words ? wv[w0 + 2] : 0ull;
                lo[u] = sh ? (a >> sh) | (b << (64 - sh)) : a;  // bits [base, base + 64)
                hi[u] = sh ? (b >> sh) | (c << (64 - sh)) : b;  // bits [base + 64, base + 128)
            }
        }
        const int valid = min(4, I.J - 4 * q);  // jobs past J are zero bytes
        for (int s = 0; s < I.S; ++s) {
            const int o = __ldg(I.sbo + s), nb = __ldg(I.bps + s);
            const unsigned M = (unsigned)__ldg(I.M + s);
            unsigned v = 0;
#pragma unroll
            for (int u = 0; u < 4; ++u)
                if (u < valid) v |= window_gene(lo[u], hi[u], o, nb, M) << (8 * u);
            reinterpret_cast<unsigned*>(dst + (size_t)s * I.Jpad)[q] = v;
        }
    }
}

__global__ void __launch_bounds__(256) k_unpack_rows(DevInst I, const unsigned long long* words,
                                                      const long long* src_idx, uint8_t* rows, long long row_stride,
                                                      const long long* dst_idx, long long n) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n) return;
    const long long src = src_idx ? src_idx[warp] : warp;
    const long long dst = dst_idx ? dst_idx[warp] : warp;
    unpack_member(I, words + src * I.words, rows + dst * row_stride, lane);
}

// ---------------------------------------------------------------------------- K3 cellular breed
constexpr int kMutChunk = 16;  // draws per lane per window of the mutation stream parse

// compute_cell (cellular.cpp:116-150) for one cell per warp.  The serial prefix (tournaments,
// crossover coin and cut points) is replayed redundantly by every lane; the mutation loop
// (one coin per gene plus one index draw per mutated gene, 148-150) is parsed warp-parallel:
// draw k of the cell stream is mix(seed + (k+1) gamma), so each lane evaluates its slice of
// the stream and a warp scan of the 2-state {coin, index} automaton assigns gene indices.
__device__ __forceinline__ unsigned long long shfl_max_u64(unsigned long long v) {
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        const unsigned long long o = __shfl_xor_sync(kFull, v, off);
        v = o > v ? o : v;
    }
    return v;
}

// Parent rows stream through K3 once (20 KB per cell); loading them without an L1 allocation keeps
// the L1 of an SM shared with a K1 CTA of the other chain for that CTA's processing-time slice.
__device__ __forceinline__ uint4 ld_row_stream(const uint4* p) {
    uint4 v;
    asm("ld.global.nc.L1::no_allocate.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
    return v;
}

// One cell, one warp: writes the child rows and returns the number of stream draws consumed.
__device__ unsigned long long breed_cell(const DevInst& I, const CellIsland& C, int cell, unsigned long long cs,
                                         const double* __restrict__ fit, const uint8_t* __restrict__ selq,
                                         uint8_t* __restrict__ child, int lane) {
    const int n = C.n;
    const int L = I.J * I.S;
    unsigned long long k = 0;
    const int npc = C.npc;
    const int* slots = C.slots + (size_t)cell * npc;

    auto tour = [&]() {  // cellular.cpp:108-112
        const int a = slots[index_of(draw(cs, k), npc)];
        const int b = slots[index_of(draw(cs, k + 1), npc)];
        k += 2;
        return fit[b] > fit[a] ? b : a;
    };
    const int p1 = tour();
    int p2 = tour();
    for (int tries = 0; p2 == p1 && tries < 8; ++tries) p2 = tour();
    if (p2 == p1) {
        for (int t = 0; t < npc; ++t)
            if (slots[t] != p1) { p2 = slots[t]; break; }
    }
    const bool crossed = coin_of(draw(cs, k++), C.thr_xr);
    int lo = 0, hi = 0;
    if (crossed) {
        const int a = index_of(draw(cs, k++), L + 1);
        int b = index_of(draw(cs, k++), L + 1);
        while (b == a) b = index_of(draw(cs, k++), L + 1);
        lo = min(a, b);
        hi = max(a, b);
    }

    const size_t block = (size_t)I.S * I.Jpad;
    FFSGA_CHECK(p1 >= 0 && p1 < n && p2 >= 0 && p2 < n, 20, p1, p2);
    FFSGA_CHECK(selq[p1] <= 1 && selq[p2] <= 1 && lo <= hi && hi <= L, 21, lo, hi);
    const uint8_t* g1 = C.genes + ((size_t)selq[p1] * n + p1) * block;
    const uint8_t* g2 = C.genes + ((size_t)selq[p2] * n + p2) * block;

    // two-point crossover on the job-major index i = j*S + s (cellular.cpp:136-146): in stage
    // row s, jobs j with lo <= j*S+s < hi, i.e. ceil((lo-s)/S) <= j < ceil((hi-s)/S), take parent 2
    const int vec_per_row = I.Jpad / 16;
    const double invS = 1.0 / (double)I.S;
    auto ceil_div_S = [&](int x) {  // ceil(x / S) for x >= 0, divide-free
        int q = (int)((double)x * invS);
        q -= (q * I.S > x) ? 1 : 0;
        q += ((q + 1) * I.S <= x) ? 1 : 0;  // q = floor(x / S)
        return q + ((q * I.S < x) ? 1 : 0);
    };
    auto byte_mask = [](int b0, int b1, int w) {  // bytes [b0, b1) of word w (bytes 4w..4w+3)
        const int l = min(max(b0 - 4 * w, 0), 4), h = min(max(b1 - 4 * w, 0), 4);
        const unsigned ml = l >= 4 ? 0u : (0xFFFFFFFFu << (8 * l));
        const unsigned mh = h >= 4 ? 0xFFFFFFFFu : ~(0xFFFFFFFFu << (8 * h));
        return ml & mh;
    };
    int s = 0, vr = lane;  // vector lane of stage row s, stepping by 32 without a divide
    while (vr >= vec_per_row && s < I.S) {
        vr -= vec_per_row;
        ++s;
    }
    for (; s < I.S;) {
        const int j0 = vr * 16;
        uint4 a = ld_row_stream(reinterpret_cast<const uint4*>(g1 + (size_t)s * I.Jpad) + vr);
        if (crossed) {
            const int jlo = lo - s <= 0 ? 0 : ceil_div_S(lo - s);
            const int jhi = hi - s <= 0 ? 0 : ceil_div_S(hi - s);
            if (jlo < j0 + 16 && jhi > j0 && jlo < jhi) {
                const uint4 b = ld_row_stream(reinterpret_cast<const uint4*>(g2 + (size_t)s * I.Jpad) + vr);
                const int b0 = jlo - j0, b1 = jhi - j0;
                unsigned m;
                m = byte_mask(b0, b1, 0);
                a.x = (a.x & ~m) | (b.x & m);
                m = byte_mask(b0, b1, 1);
                a.y = (a.y & ~m) | (b.y & m);
                m = byte_mask(b0, b1, 2);
                a.z = (a.z & ~m) | (b.z & m);
                m = byte_mask(b0, b1, 3);
                a.w = (a.w & ~m) | (b.w & m);
            }
        }
        reinterpret_cast<uint4*>(child + (size_t)s * I.Jpad)[vr] = a;
        vr += 32;
        while (vr >= vec_per_row && s < I.S) {
            vr -= vec_per_row;
            ++s;
        }
    }
    __syncwarp();

    // mutation (cellular.cpp:148-150)
    const unsigned long long thr = C.thr_mu;
    const bool always = thr >= (1ull << 53);                  // p = 1: every coin is true
    const unsigned long long ulim = always ? 0ull : (thr << 11);  // (u>>11) < thr  <=>  u < thr<<11
    unsigned long long pos = k;
    unsigned long long end = k;
    int coins_before = 0;
    bool st_coin = true;
    while (coins_before < L || (coins_before == L && !st_coin)) {
        const unsigned long long p0 = pos + (unsigned long long)lane * kMutChunk;
        unsigned tb = 0;  // bit t: draw t would be a true coin
#pragma unroll
        for (int t = 0; t < kMutChunk; ++t) {
            const unsigned long long u = draw(cs, p0 + t);
            tb |= ((always || u < ulim) ? 1u : 0u) << t;
        }
        // which draws of this lane's slice are coins, for both entry states.  A true coin makes
        // the next draw an index draw, which cannot itself start another -- the escape rule of
        // backslashes in a string -- so the index (escaped) positions follow bit-parallel from
        // the carry trick for runs of escapes (add on odd run starts, flip every other bit).
        static_assert(kMutChunk == 16, "the escape masks below are written for 16-draw slices");
        auto coins = [tb](unsigned first_is_index, unsigned& cm, int& next_is_coin) {
            const unsigned bs = tb & ~first_is_index;                    // an index draw escapes nothing
            const unsigned follows = (bs << 1) | first_is_index;
            const unsigned odd_starts = bs & ~0x5555u & ~follows;
            const unsigned flip = (odd_starts + bs) << 1;
            const unsigned esc = (0x5555u ^ flip) & follows & 0xFFFFu;    // index draws
            cm = ~esc & 0xFFFFu;
            next_is_coin = ((cm & tb) >> 15) & 1u ? 0 : 1;
        };
        unsigned cm1, cm0;
        int f1, f0;
        coins(0u, cm1, f1);
        coins(1u, cm0, f0);
        const int c1 = __popc(cm1), c0 = __popc(cm0);
        // inclusive scan (composition) over lanes
        int F0 = f0, F1 = f1, C0 = c0, C1 = c1;
#pragma unroll
        for (int off = 1; off < 32; off <<= 1) {
            const int pF0 = __shfl_up_sync(kFull, F0, off);
            const int pF1 = __shfl_up_sync(kFull, F1, off);
            const int pC0 = __shfl_up_sync(kFull, C0, off);
            const int pC1 = __shfl_up_sync(kFull, C1, off);
            if (lane >= off) {
                // new(x) = me(prev(x))
                const int nF0 = pF0 ? F1 : F0, nC0 = pC0 + (pF0 ? C1 : C0);
                const int nF1 = pF1 ? F1 : F0, nC1 = pC1 + (pF1 ? C1 : C0);
                F0 = nF0; C0 = nC0; F1 = nF1; C1 = nC1;
            }
        }
        // exclusive prefix for this lane given the window entry state
        const int eF0 = __shfl_up_sync(kFull, F0, 1), eF1 = __shfl_up_sync(kFull, F1, 1);
        const int eC0 = __shfl_up_sync(kFull, C0, 1), eC1 = __shfl_up_sync(kFull, C1, 1);
        int st, g;
        if (lane == 0) {
            st = st_coin;
            g = coins_before;
        } else {
            st = st_coin ? eF1 : eF0;
            g = coins_before + (st_coin ? eC1 : eC0);
        }
        const unsigned cm = st ? cm1 : cm0;  // coin draws of the slice: coin #r is gene g + r
        // gene L-1's coin ends the loop's draws (plus its index draw when true)
        const int ncoin = __popc(cm);
        if (g <= L - 1 && L - 1 < g + ncoin) {
            const int t = (int)__fns(cm, 0, L - g);  // (L-1-g)+1-th set bit
            end = p0 + t + 1 + ((tb >> t) & 1u);
        }
        // index draws: right after a true coin (and draw 0 when the slice starts inside a pair)
        unsigned im = ((cm & tb) << 1) & ((1u << kMutChunk) - 1u);
        if (!st) im |= 1u;
        while (im) {  // rare (mutation rate), divergent but short
            const int t = __ffs(im) - 1;
            im &= im - 1u;
            const int gene = g + __popc(cm & ((1u << t) - 1u)) - 1;
            if (gene < L) {
                int j = (int)((double)gene * invS);  // gene / S without an integer divide
                j -= (j * I.S > gene) ? 1 : 0;
                j += ((j + 1) * I.S <= gene) ? 1 : 0;
                const int s = gene - j * I.S;
                FFSGA_CHECK(j >= 0 && j < I.J && s >= 0 && s < I.S, 22, gene, cell);
                child[(size_t)s * I.Jpad + j] = (uint8_t)index_of(draw(cs, p0 + t), __ldg(I.M + s));
            }
        }
        const int lF0 = __shfl_sync(kFull, F0, 31), lF1 = __shfl_sync(kFull, F1, 31);
        const int lC0 = __shfl_sync(kFull, C0, 31), lC1 = __shfl_sync(kFull, C1, 31);
        coins_before += st_coin ? lC1 : lC0;
        st_coin = st_coin ? lF1 : lF0;
        pos += 32ull * kMutChunk;
    }
    return shfl_max_u64(end);
}

// compute_cell (cellular.cpp:116-150) for one cell per warp.  The serial prefix (tournaments,
// crossover coin and cut points) is replayed redundantly by every lane; the mutation loop
// (one coin per gene plus one index draw per mutated gene, 148-150) is parsed warp-parallel:
// draw k of the cell stream is mix(seed + (k+1) gamma), so each lane evaluates its slice of
// the stream and a warp scan of the 2-state {coin, index} automaton assigns gene indices.
__global__ void __launch_bounds__(256) k_cell_breed(DevInst I, const CellIsland* __restrict__ isl,
                                                     int n_islands, long long n_cells, WorkList wl) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n_cells) return;
    int ii = 0;
    while (ii + 1 < n_islands && isl[ii + 1].cell0 <= warp) ++ii;
    const CellIsland& C = isl[ii];
    const int cell = (int)(warp - C.cell0);
    const int n = C.n;
    const unsigned long long gen = C.st->gen;
    const int q = (int)(gen & 1ull);
    const uint8_t* selq = C.sel + (size_t)q * n;
    const unsigned long long gen_seed = derive_seed(C.seed, gen + 1ull);  // cellular.cpp:167
    const unsigned long long cs = derive_seed(gen_seed, (unsigned long long)cell);  // :171
    uint8_t* child = C.genes + ((size_t)(1 - selq[cell]) * n + cell) * ((size_t)I.S * I.Jpad);
    breed_cell(I, C, cell, cs, C.fit + (size_t)q * n, selq, child, lane);
    if (lane == 0) wl.ptrs[C.item0 + cell] = child;
}

// cell_candidate (cellular.cpp:157-162) on an explicit stream: child rows into `out`.
__global__ void k_cell_candidate(DevInst I, CellIsland C, int cell, unsigned long long cs, int q, uint8_t* out,
                                 unsigned long long* draws) {
    const int lane = threadIdx.x & 31;
    const unsigned long long used =
        breed_cell(I, C, cell, cs, C.fit + (size_t)q * C.n, C.sel + (size_t)q * C.n, out, lane);
    if (lane == 0) *draws = used;
}

// ---------------------------------------------------------------------------- K4 pseudo breed
// pair_step (pseudo.cpp:11-29) for one pair per warp: coin, then one mask word per 64 bits,
// children written in place; crossed members are appended to the evaluation work list with
// their gene rows (bits_to_int, chromosome.cpp:44-59) in the island's row storage.
__global__ void __launch_bounds__(256) k_pseudo_breed(DevInst I, const PseudoIsland* __restrict__ isl,
                                                       int n_islands, long long n_pairs, WorkList wl) {
    const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= n_pairs) return;
    int ii = 0;
    while (ii + 1 < n_islands && isl[ii + 1].pair0 <= warp) ++ii;
    const PseudoIsland& P = isl[ii];
    const int pair = (int)(warp - P.pair0);
    const unsigned long long gen = P.st->gen;
    const unsigned long long gen_seed = derive_seed(P.seed, gen + 1ull);  // pseudo.cpp:61
    const unsigned long long ps = derive_seed(gen_seed, (unsigned long long)pair);  // :68
    const bool crossed = coin_of(draw(ps, 0), P.thr_xr);
    if (!crossed) {
        if (lane == 0) {
            P.mslot[2 * pair] = -1;
            P.mslot[2 * pair + 1] = -1;
        }
        return;
    }
    unsigned long long* A = P.words + (size_t)(2 * pair) * I.words;
    unsigned long long* B = A + I.words;
    for (int w = lane; w < I.words; w += 32) {
        const unsigned long long msk = draw(ps, 1ull + (unsigned long long)w);
        const unsigned long long a = A[w], b = B[w];
        A[w] = (a & msk) | (b & ~msk);
        B[w] = (b & msk) | (a & ~msk);
    }
    long long slot = 0;
    if (lane == 0) slot = atomicAdd(reinterpret_cast<unsigned long long*>(wl.count), 2ull);
    slot = __shfl_sync(kFull, slot, 0);
    __syncwarp();
    const size_t block = (size_t)I.S * I.Jpad;
    uint8_t* r1 = P.rows + (size_t)(2 * pair) * block;  // the island's own row storage
    uint8_t* r2 = r1 + block;
    unpack_member(I, A, r1, lane);
    unpack_member(I, B, r2, lane);
    if (lane == 0) {
        wl.ptrs[slot] = r1;
        wl.ptrs[slot + 1] = r2;
        P.mslot[2 * pair] = slot;
        P.mslot[2 * pair + 1] = slot + 1;
    }
}

__global__ void k_gen_begin(long long* count, long long v) { *count = v; }

// ---------------------------------------------------------------------------- K6 commit
struct Best {
    double f;
    int i;
};
__device__ __forceinline__ Best better(Best a, Best b) {  // first index of the max
    if (b.f > a.f || (b.f == a.f && b.i < a.i)) return b;
    return a;
}

__device__ Best block_best(Best v) {
    __shared__ double sf[32];
    __shared__ int si[32];
    const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
        Best o{__shfl_xor_sync(kFull, v.f, off), __shfl_xor_sync(kFull, v.i, off)};
        v = better(v, o);
    }
    __syncthreads();
    if (lane == 0) { sf[wid] = v.f; si[wid] = v.i; }
    __syncthreads();
    const int nw = (blockDim.x + 31) >> 5;
    if (wid == 0) {
        Best x = lane < nw ? Best{sf[lane], si[lane]} : Best{-dinf(), 0x7FFFFFFF};
#pragma unroll
        for (int off = 16; off > 0; off >>= 1) {
            Best o{__shfl_xor_sync(kFull, x.f, off), __shfl_xor_sync(kFull, x.i, off)};
            x = better(x, o);
        }
        if (lane == 0) { sf[0] = x.f; si[0] = x.i; }
    }
    __syncthreads();
    return Best{sf[0], si[0]};
}

// One CTA per island.  Cellular: strict-improvement replacement into the next parity buffers
// (cellular.cpp:153,175-180); pseudo: unconditional replacement + archive scan in pair order
// (pseudo.cpp:74-87).  Then best_index (first max) and the per-generation trace value
// (solver.cpp:113,121), and ++generation.
__global__ void __launch_bounds__(1024) k_commit(DevInst I, const CellIsland* __restrict__ cells, int nc,
                                                  const PseudoIsland* __restrict__ pseudo, int np, WorkList wl,
                                                  int mode) {
    // mode 0: refresh best only; 1: commit one generation; 2: pseudo init (archive over all)
    const int advance = mode == 1;
    const int b = blockIdx.x;
    if (advance && b == 0 && threadIdx.x == 0 && wl.total) atomicAdd(wl.total, (unsigned long long)*wl.count);
    if (b < nc) {
        const CellIsland& C = cells[b];
        const int n = C.n;
        const unsigned long long gen = C.st->gen;
        const int q = (int)(gen & 1ull);
        const int nq = advance ? 1 - q : q;
        Best best{-dinf(), 0x7FFFFFFF};
        for (int c = threadIdx.x; c < n; c += blockDim.x) {
            double f = C.fit[(size_t)q * n + c];
            double o = C.obj[(size_t)q * n + c];
            uint8_t s = C.sel[(size_t)q * n + c];
            if (advance) {
                const double cf = wl.fit[C.item0 + c];
                if (cf > f) {
                    f = cf;
                    o = wl.obj[C.item0 + c];
                    s = (uint8_t)(1 - s);
                }
                C.fit[(size_t)nq * n + c] = f;
                C.obj[(size_t)nq * n + c] = o;
                C.sel[(size_t)nq * n + c] = s;
            }
            best = better(best, Best{f, c});
        }
        best = block_best(best);
        if (threadIdx.x == 0) {
            IslandState* st = C.st;
            st->best_idx = best.i;
            st->best_fit = best.f;
            st->best_obj = C.obj[(size_t)nq * n + best.i];
            if (advance) {
                C.trace[gen - st->seg_start] = st->best_obj;
                st->gen = gen + 1ull;
            }
        }
        return;
    }
    const PseudoIsland& P = pseudo[b - nc];
    const int n = P.n;
    Best live{-dinf(), 0x7FFFFFFF}, changed{-dinf(), 0x7FFFFFFF};
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double f = P.fit[i];
        if (advance) {
            const long long k = P.mslot[i];
            if (k >= 0) {
                f = wl.fit[k];
                P.fit[i] = f;
                P.obj[i] = wl.obj[k];
                changed = better(changed, Best{f, i});
            }
        } else if (mode == 2) {
            changed = better(changed, Best{f, i});
        }
        live = better(live, Best{f, i});
    }
    live = block_best(live);
    changed = block_best(changed);
    IslandState* st = P.st;
    const bool take = changed.i != 0x7FFFFFFF && changed.f > st->arch_fit;
    if (take)
        for (int w = threadIdx.x; w < I.words; w += blockDim.x)
            P.archive[w] = P.words[(size_t)changed.i * I.words + w];
    __syncthreads();
    if (threadIdx.x == 0) {
        if (take) {
            st->arch_fit = changed.f;
            st->arch_obj = P.obj[changed.i];
        }
        st->best_idx = live.i;
        st->best_fit = live.f;
        st->best_obj = P.obj[live.i];
        if (advance) {
            const unsigned long long gen = st->gen;
            P.trace[gen - st->seg_start] = st->arch_obj;
            st->gen = gen + 1ull;
        }
    }
}

// ---------------------------------------------------------------------------- K5 migration
__global__ void k_fill_seq(long long* idx, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) idx[i] = i;
}

__global__ void k_sort_keys(const double* fit, double* keys, long long n) {
    const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const double f = fit[i];
        keys[i] = (f == 0.0) ? 0.0 : f;  // canonical +0.0: radix order must match == ties
    }
}

// Migrant packets (cross-device migration, islands.py): k migrants as they leave their island,
// [fit[k] fp64][obj[k] fp64][payload], payload = k stage-major gene rows of S*Jpad bytes (from a
// cellular island) or k packed members of W u64 words (from a pseudo island).  An exporter
// writes one on its own GPU, the bytes travel over NCCL / NVLink, the importer installs them
// with the same kernels as a device-local migration (migration.cpp:47-69).

// k best cells (sort_island order) -> packet rows + fit/obj
__global__ void k_export_cell(DevInst I, CellIsland C, const long long* best_c, int k, int parity, uint8_t* rows,
                              double* fo) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= k) return;
    const long long src = best_c[warp];
    const size_t block = (size_t)I.S * I.Jpad;
    const uint4* r = reinterpret_cast<const uint4*>(C.genes + ((size_t)C.sel[(size_t)parity * C.n + src] * C.n + src) * block);
    uint4* out = reinterpret_cast<uint4*>(rows + (size_t)warp * block);
    for (size_t v = lane; v < block / 16; v += 32) out[v] = r[v];
    if (lane == 0) {
        fo[warp] = C.fit[(size_t)parity * C.n + src];
        fo[k + warp] = C.obj[(size_t)parity * C.n + src];
    }
}

// k best members (sort_island order) -> packet words + fit/obj
__global__ void k_export_pseudo(DevInst I, PseudoIsland P, const long long* best_p, int k, unsigned long long* words,
                                double* fo) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= k) return;
    const long long src = best_p[warp];
    for (int w = lane; w < I.words; w += 32) words[(size_t)warp * I.words + w] = P.words[src * I.words + w];
    if (lane == 0) {
        fo[warp] = P.fit[src];
        fo[k + warp] = P.obj[src];
    }
}

// cellular -> pseudo (migration.cpp:47-57): best[i] of the cellular island (or row i of a packet)
// lands on worst[N-1-i] of the pseudo island, converted with int_to_bits; the archive absorbs
// the installs in order (pseudo.cpp:98-104).
__global__ void k_migrate_c2p(DevInst I, CellIsland C, PseudoIsland P, const long long* best_c,
                              const long long* worst_p, int k, int parity, const uint16_t* bit_stage,
                              const uint8_t* pk_rows, const double* pk_fo) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= k) return;
    const long long dst = worst_p[P.n - 1 - warp];
    const size_t block = (size_t)I.S * I.Jpad;
    const long long src = pk_rows ? warp : best_c[warp];
    const uint8_t* r = pk_rows ? pk_rows + (size_t)warp * block
                               : C.genes + ((size_t)C.sel[(size_t)parity * C.n + src] * C.n + src) * block;
    for (int w = lane; w < I.words; w += 32) P.words[dst * I.words + w] = pack_word(I, r, w, bit_stage);
    if (lane == 0) {
        P.fit[dst] = pk_rows ? pk_fo[warp] : C.fit[(size_t)parity * C.n + src];
        P.obj[dst] = pk_rows ? pk_fo[k + warp] : C.obj[(size_t)parity * C.n + src];
    }
}

__global__ void k_migrate_archive(DevInst I, PseudoIsland P, const long long* worst_p, int k) {
    // consider_for_archive over the installs in order: the first strict maximum wins
    Best b{-dinf(), 0x7FFFFFFF};
    for (int i = threadIdx.x; i < k; i += blockDim.x) b = better(b, Best{P.fit[worst_p[P.n - 1 - i]], i});
    b = block_best(b);
    IslandState* st = P.st;
    const bool take = b.i != 0x7FFFFFFF && b.f > st->arch_fit;
    __syncthreads();
    if (take) {
        const long long dst = worst_p[P.n - 1 - b.i];
        for (int w = threadIdx.x; w < I.words; w += blockDim.x) P.archive[w] = P.words[dst * I.words + w];
        if (threadIdx.x == 0) {
            st->arch_fit = b.f;
            st->arch_obj = P.obj[dst];
        }
    }
}

// pseudo -> cellular (migration.cpp:59-69): bits_to_int into the cell's live storage slot.
__global__ void k_migrate_p2c(DevInst I, PseudoIsland P, CellIsland C, const long long* best_p,
                              const long long* worst_c, int k, int parity, const unsigned long long* pk_words,
                              const double* pk_fo) {
    const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int lane = threadIdx.x & 31;
    if (warp >= k) return;
    const long long dst = worst_c[C.n - 1 - warp];
    const size_t block = (size_t)I.S * I.Jpad;
    uint8_t* r = C.genes + ((size_t)C.sel[(size_t)parity * C.n + dst] * C.n + dst) * block;
    const long long src = pk_words ? warp : best_p[warp];
    unpack_member(I, (pk_words ? pk_words : P.words) + src * I.words, r, lane);
    if (lane == 0) {
        C.fit[(size_t)parity * C.n + dst] = pk_words ? pk_fo[warp] : P.fit[src];
        C.obj[(size_t)parity * C.n + dst] = pk_words ? pk_fo[k + warp] : P.obj[src];
    }
}

inline unsigned blocks_for(long long threads, int per_block) {
    return (unsigned)((threads + per_block - 1) / per_block);
}

template <int G>
int eval_config_g(const DevInst& I, int sm_count, int warps_cap, EvalConfig* cfg) {
    (void)sm_count;
    cfg->G = G;
    cfg->gl = group_layout(I.J, I.Jpad, G);
    cfg->bl = bucket_layout(I.J, I.Jpad, G, I.bshift);
    if (I.algo == 1) cfg->gl.bytes = cfg->bl.bytes;  // bytes per group of the decoder in use
    const int max_smem = 227 * 1024;
    const size_t per_warp = (size_t)(32 / G) * cfg->gl.bytes;
    int warps = (int)std::min<size_t>(warps_cap > 0 ? warps_cap : 16, max_smem / per_warp);
    if (warps < 1) return -1;
    // Leave at least ~27 KB of the unified L1 to the stage's processing-time slice when that
    // costs no more than one warp: the pop loop's procT loads then mostly hit L1 (500x20: one
    // 8-warp CTA 9.86 M evals/s, 9 warps 9.34, two 4-warp CTAs 9.37 -- two CTAs pull two
    // stage slices through the same L1).
    const int pref = (int)((200 * 1024) / per_warp);
    if (pref >= 1) warps = std::min(warps, pref);
    cfg->warps = warps;
    cfg->groups_per_cta = 32 * warps / G;
    cfg->smem = (size_t)cfg->groups_per_cta * cfg->gl.bytes;
    // Pop pipeline depth: three pops in flight for large instances (1000x20: +5 %), two
    // otherwise (500x20: the third slot costs 1.5 %; 100x10: -32 %, registers bind there)
    cfg->depth = 2;
    const void* k0 = I.algo == 1 ? (const void*)k_eval_bkt<G, false> : (const void*)k_eval<G, false, 2, false>;
    if constexpr (G <= 8) {
        if (I.algo != 1 && I.pk_bits) k0 = (const void*)k_eval<G, false, 2, true>;
    }
    if constexpr (G == 8) {
        const char* dv = getenv("FFSGA_EVAL_DEPTH");  // experiments: 2, 3 or 4
        // measured thresholds (C5 shapes, M in [2, 8]): the 4-deep body wins from J = 300 on
        // (256x10: 44.4 vs 32.0 M evals/s for the 2-deep body; 300x10 and 256x20: equal)
        const int want = dv ? atoi(dv) : (I.J >= 1000 ? 3 : (I.J >= 300 ? 4 : 2));
        if (I.algo != 1 && want == 3) {
            cfg->depth = 3;
            k0 = I.pk_bits ? (const void*)k_eval<8, false, 3, true> : (const void*)k_eval<8, false, 3, false>;
        } else if (I.algo != 1 && want == 4) {
            cfg->depth = 4;
            k0 = I.pk_bits ? (const void*)k_eval<8, false, 4, true> : (const void*)k_eval<8, false, 4, false>;
        }
    }
    const void* k1 = I.algo == 1 ? (const void*)k_eval_bkt<G, true> : (const void*)k_eval<G, true, 2, false>;
    // the opt-in ceiling, not this config's size: configs of other instances (other J) and the
    // joint-step config share the kernel's attribute
    cudaError_t e = cudaFuncSetAttribute(k0, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
    if (e != cudaSuccess) return -2;
    e = cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, max_smem);
    if (e != cudaSuccess) return -2;
    int occ = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k0, 32 * warps, cfg->smem);
    if (e != cudaSuccess || occ < 1) return -2;
    if (const char* v = getenv("FFSGA_EVAL_CTAS_PER_SM")) occ = std::max(1, std::min(occ, atoi(v)));  // experiments
    cfg->blocks_per_sm = occ;
    return 0;
}

template <int G>
cudaError_t launch_eval_g(const DevInst& I, const EvalConfig& cfg, const EvalItems& W, long long max_items,
                          int sm_count, bool schedule, cudaStream_t st) {
    if (max_items <= 0 && !W.n_dev) return cudaSuccess;  // nothing to decode (an empty batch)
    long long blocks = (max_items + cfg.groups_per_cta - 1) / cfg.groups_per_cta;
    const long long cap = (long long)cfg.blocks_per_sm * sm_count;
    if (blocks > cap) blocks = cap;
    if (blocks < 1) blocks = 1;
    if (W.deal && I.algo != 1 && !schedule && blocks < sm_count) {
        // A small launch that owns the GPU (one island, C1/C2): full CTAs would leave most SMs
        // idle, so spread the items over up to one CTA per SM with fewer warps each -- a
        // chromosome on a thinly filled SM decodes faster (less issue contention per pop).
        constexpr int per_warp = 32 / G;
        const long long want = (max_items + sm_count - 1) / sm_count;
        const int gpc = (int)(((want + per_warp - 1) / per_warp) * per_warp);
        if (gpc < cfg.groups_per_cta) {
            EvalConfig c = cfg;
            c.groups_per_cta = gpc;
            c.warps = gpc / per_warp;
            c.smem = (size_t)gpc * cfg.gl.bytes;
            c.blocks_per_sm = 1;
            return launch_eval_g<G>(I, c, W, max_items, sm_count, schedule, st);
        }
    }
    if (I.algo == 1) {
        if (schedule)
            k_eval_bkt<G, true><<<(unsigned)blocks, 32 * cfg.warps, cfg.smem, st>>>(I, W, cfg.groups_per_cta, cfg.bl);
        else
            k_eval_bkt<G, false><<<(unsigned)blocks, 32 * cfg.warps, cfg.smem, st>>>(I, W, cfg.groups_per_cta, cfg.bl);
    } else if (schedule) {
        k_eval<G, true, 2, false><<<(unsigned)blocks, 32 * cfg.warps, cfg.smem, st>>>(I, W, cfg.groups_per_cta, cfg.gl);
    } else {
        const dim3 grid((unsigned)blocks), block(32 * cfg.warps);
        if constexpr (G == 8) {
            if (cfg.depth == 3) {
                if (I.pk_bits)
                    k_eval<8, false, 3, true><<<grid, block, cfg.smem, st>>>(I, W, cfg.groups_per_cta, cfg.gl);
                else
                    k_eval<8, false, 3, false><<<grid, block, cfg.smem, st>>>(I, W, cfg.groups_per_cta, cfg.gl);
                return cudaGetLastError();
            }
            if (cfg.depth == 4) {
                if (I.pk_bits)
                    k_eval<8, false, 4, true><<<grid, block, cfg.smem, st>>>(I, W, cfg.groups_per_cta, cfg.gl);
                else
                    k_eval<8, false, 4, false><<<grid, block, cfg.smem, st>>>(I, W, cfg.groups_per_cta, cfg.gl);
                return cudaGetLastError();
            }
        }
        if constexpr (G <= 8) {
            if (I.pk_bits) {
                k_eval<G, false, 2, true><<<grid, block, cfg.smem, st>>>(I, W, cfg.groups_per_cta, cfg.gl);
                return cudaGetLastError();
            }
        }
        k_eval<G, false, 2, false><<<grid, block, cfg.smem, st>>>(I, W, cfg.groups_per_cta, cfg.gl);
    }
    return cudaGetLastError();
}

}  // namespace

int eval_config(const DevInst& I, int sm_count, int warps_cap, EvalConfig* cfg) {
    // The smallest group that covers the widest stage; when a warp of such groups does not fit
    // shared memory (large J), wider groups put fewer chromosomes in a warp (idle lanes) so that
    // one chromosome may use up to a whole CTA's shared memory.
    int rc = -3;
    const int gmin = getenv("FFSGA_EVAL_G") ? atoi(getenv("FFSGA_EVAL_G")) : 0;  // experiments
    if (I.maxM <= 4 && gmin <= 4 && (rc = eval_config_g<4>(I, sm_count, warps_cap, cfg)) != -1) return rc;
    if (I.maxM <= 8 && (rc = eval_config_g<8>(I, sm_count, warps_cap, cfg)) != -1) return rc;
    if (I.maxM <= 16 && (rc = eval_config_g<16>(I, sm_count, warps_cap, cfg)) != -1) return rc;
    if (I.maxM <= 32) return eval_config_g<32>(I, sm_count, warps_cap, cfg);
    return rc;
}

cudaError_t launch_eval(const DevInst& I, const EvalConfig& cfg, const EvalItems& W, long long max_items,
                        int sm_count, bool schedule, cudaStream_t st) {
    switch (cfg.G) {
        case 4: return launch_eval_g<4>(I, cfg, W, max_items, sm_count, schedule, st);
        case 8: return launch_eval_g<8>(I, cfg, W, max_items, sm_count, schedule, st);
        case 16: return launch_eval_g<16>(I, cfg, W, max_items, sm_count, schedule, st);
        case 32: return launch_eval_g<32>(I, cfg, W, max_items, sm_count, schedule, st);
    }
    return cudaErrorInvalidValue;
}

cudaError_t launch_random_rows(const DevInst& I, uint8_t* out, long long stride, long long n,
                               unsigned long long base, long long first, bool per_item, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_random_rows<<<blocks_for(n * 32, 256), 256, 0, st>>>(I, out, stride, n, base, first, per_item ? 1 : 0);
    return cudaGetLastError();
}

cudaError_t launch_pack_bits(const DevInst& I, const uint8_t* rows, long long row_stride, const long long* src_idx,
                             unsigned long long* words, const long long* dst_idx, long long n, bool with_complement,
                             const uint16_t* bit_stage, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_pack_bits<<<blocks_for(n * 32, 256), 256, 0, st>>>(I, rows, row_stride, src_idx, words, dst_idx, n,
                                                        with_complement ? 1 : 0, bit_stage);
    return cudaGetLastError();
}

cudaError_t launch_unpack_rows(const DevInst& I, const unsigned long long* words, const long long* src_idx,
                               uint8_t* rows, long long row_stride, const long long* dst_idx, long long n,
                               cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_unpack_rows<<<blocks_for(n * 32, 256), 256, 0, st>>>(I, words, src_idx, rows, row_stride, dst_idx, n);
    return cudaGetLastError();
}

cudaError_t launch_rows_from_int(const DevInst& I, const int32_t* gi, const uint8_t* gu, uint8_t* rows, long long n,
                                 cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_rows_from_int<<<blocks_for(n * 32, 256), 256, 0, st>>>(I, gi, gu, rows, n);
    return cudaGetLastError();
}

cudaError_t launch_rows_to_int(const DevInst& I, const uint8_t* rows, long long row_stride, const long long* src_idx,
                               int32_t* out, long long n, cudaStream_t st) {
    if (n <= 0) return cudaSuccess;
    k_rows_to_int<<<blocks_for(n * 32, 256), 256, 0, st>>>(I, rows, row_stride, src_idx, out, n);
    return cudaGetLastError();
}

cudaError_t launch_breed(const DevInst& I, const CellIsland* cells_dev, int nc, long long n_cells,
                         const PseudoIsland* pseudo_dev, int np, long long n_pairs, const WorkList& wl,
                         cudaStream_t st) {
    k_gen_begin<<<1, 1, 0, st>>>(wl.count, nc > 0 ? n_cells : 0);
    if (n_cells > 0) k_cell_breed<<<blocks_for(n_cells * 32, 256), 256, 0, st>>>(I, cells_dev, nc, n_cells, wl);
    if (n_pairs > 0) k_pseudo_breed<<<blocks_for(n_pairs * 32, 256), 256, 0, st>>>(I, pseudo_dev, np, n_pairs, wl);
    return cudaGetLastError();
}

cudaError_t launch_commit(const DevInst& I, const CellIsland* cells_dev, int nc, const PseudoIsland* pseudo_dev,
                          int np, const WorkList& wl, cudaStream_t st) {
    k_commit<<<nc + np, 1024, 0, st>>>(I, cells_dev, nc, pseudo_dev, np, wl, 1);
    return cudaGetLastError();
}

cudaError_t launch_island_stats(const DevInst& I, const CellIsland* cells_dev, int nc, const PseudoIsland* pseudo_dev,
                                int np, int mode, cudaStream_t st) {
    if (nc + np == 0) return cudaSuccess;
    WorkList wl{};
    k_commit<<<nc + np, 1024, 0, st>>>(I, cells_dev, nc, pseudo_dev, np, wl, mode);
    return cudaGetLastError();
}

size_t sort_temp_bytes(long long n) {
    size_t bytes = 0;
    cub::DeviceRadixSort::SortPairsDescending(nullptr, bytes, (const double*)nullptr, (double*)nullptr,
                                              (const long long*)nullptr, (long long*)nullptr, (int)n);
    return bytes;
}

cudaError_t launch_sort_desc(const double* fit, long long n, double* keys_tmp, double* keys_out, long long* idx_in,
                             long long* idx_out, void* temp, size_t temp_bytes, cudaStream_t st) {
    k_sort_keys<<<blocks_for(n, 256), 256, 0, st>>>(fit, keys_tmp, n);
    k_fill_seq<<<blocks_for(n, 256), 256, 0, st>>>(idx_in, n);
    // stable radix sort: fitness descending, equal keys keep ascending index (sort_island,
    // cellular.cpp:29-36)
    return cub::DeviceRadixSort::SortPairsDescending(temp, temp_bytes, keys_tmp, keys_out, idx_in, idx_out, (int)n,
                                                     0, 64, st);
}

cudaError_t launch_migrate_c2p(const DevInst& I, const CellIsland& c, const PseudoIsland& p, const long long* best_c,
                               const long long* worst_p, int k, int parity, const uint16_t* bit_stage,
                               cudaStream_t st, const uint8_t* pk_rows, const double* pk_fo) {
    if (k <= 0) return cudaSuccess;
    k_migrate_c2p<<<blocks_for((long long)k * 32, 256), 256, 0, st>>>(I, c, p, best_c, worst_p, k, parity, bit_stage,
                                                                       pk_rows, pk_fo);
    k_migrate_archive<<<1, 1024, 0, st>>>(I, p, worst_p, k);
    return cudaGetLastError();
}

cudaError_t launch_migrate_p2c(const DevInst& I, const PseudoIsland& p, const CellIsland& c, const long long* best_p,
                               const long long* worst_c, int k, int parity, cudaStream_t st,
                               const unsigned long long* pk_words, const double* pk_fo) {
    if (k <= 0) return cudaSuccess;
    k_migrate_p2c<<<blocks_for((long long)k * 32, 256), 256, 0, st>>>(I, p, c, best_p, worst_c, k, parity, pk_words,
                                                                       pk_fo);
    return cudaGetLastError();
}

cudaError_t launch_export_cell(const DevInst& I, const CellIsland& c, const long long* best_c, int k, int parity,
                               uint8_t* rows, double* fo, cudaStream_t st) {
    if (k <= 0) return cudaSuccess;
    k_export_cell<<<blocks_for((long long)k * 32, 256), 256, 0, st>>>(I, c, best_c, k, parity, rows, fo);
    return cudaGetLastError();
}

cudaError_t launch_export_pseudo(const DevInst& I, const PseudoIsland& p, const long long* best_p, int k,
                                 unsigned long long* words, double* fo, cudaStream_t st) {
    if (k <= 0) return cudaSuccess;
    k_export_pseudo<<<blocks_for((long long)k * 32, 256), 256, 0, st>>>(I, p, best_p, k, words, fo);
    return cudaGetLastError();
}

cudaError_t launch_cell_candidate(const DevInst& I, const CellIsland& c, int cell, unsigned long long stream_seed,
                                  int parity, uint8_t* out, unsigned long long* draws, cudaStream_t st) {
    k_cell_candidate<<<1, 32, 0, st>>>(I, c, cell, stream_seed, parity, out, draws);
    return cudaGetLastError();
}

// checked build: the first failed device check (0 = none) and reset; -1 in a normal build
cudaError_t checked_status(long long* status, bool reset) {
#ifdef FFSGA_CHECKED
    unsigned long long v = 0;
    cudaError_t e = cudaMemcpyFromSymbol(&v, g_check_fail, sizeof(v));
    if (e != cudaSuccess) return e;
    *status = (long long)v;
    if (reset) {
        v = 0;
        return cudaMemcpyToSymbol(g_check_fail, &v, sizeof(v));
    }
    return cudaSuccess;
#else
    (void)reset;
    *status = -1;
    return cudaSuccess;
#endif
}

cudaError_t launch_fill_seq(long long* idx, long long n, cudaStream_t st) {
    k_fill_seq<<<blocks_for(n, 256), 256, 0, st>>>(idx, n);
    return cudaGetLastError();
}

}  // namespace ffsga_dev
