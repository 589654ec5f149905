// launch.h -- POD descriptors shared by the kernels (kernels.cu) and the C-ABI (capi.cu).
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include "device.cuh"

namespace ffsga_dev {

// Batch of chromosomes for the decoder (K1 / K7).
struct EvalItems {
    const long long* n_dev;        // item count on device (joint GA step) or nullptr
    long long n;                   // item count (plus *n_dev when set)
    const uint8_t* base;           // implicit rows: base + i * stride
    long long stride;
    const uint8_t* const* ptrs;    // explicit per-item row blocks (GA work list) or nullptr
    double* obj;
    double* fit;
    double* mk;                    // optional
    double* td;                    // optional
    unsigned long long* err;       // optional: min over (item<<32 | stage<<16 | job)
    int* smachine;                 // K7 schedule of item 0 (job-major [j*S+s])
    double* sstart;
    double* scomp;
    int deal;                      // 1: items round-robin over CTAs (launch owns the GPU)
};

struct IslandState {
    unsigned long long gen;        // generations completed (reference generation_)
    unsigned long long seg_start;  // generation at the start of the current step() call
    int best_idx;                  // first index of the max fitness (live population)
    int pad;
    double best_fit, best_obj;
    double arch_fit, arch_obj;     // pseudo archive (pseudo.hpp:78-80)
};

struct CellIsland {
    int n, width, height, npc;
    const int* slots;              // [n*npc] neighbor slots in reference order (cellular.cpp:12-27)
    uint8_t* genes;                // [2][n][S*Jpad] two storage slots per cell
    uint8_t* sel;                  // [2][n] storage slot of each cell, by generation parity
    double* fit;                   // [2][n]
    double* obj;                   // [2][n]
    unsigned long long seed;
    unsigned long long thr_xr, thr_mu;
    IslandState* st;
    double* trace;                 // [trace_cap]
    long long item0;               // first work item of this island's cells
    long long cell0;               // first global cell id
};

struct PseudoIsland {
    int n;                         // members (2 per pair)
    int pad;
    unsigned long long* words;     // [n][W]
    double* fit;                   // [n]
    double* obj;                   // [n]
    long long* mslot;              // [n] work item of a crossed member this generation, or -1
    uint8_t* rows;                 // [n][S*Jpad] gene rows of the members crossed this generation
    unsigned long long* archive;   // [W]
    unsigned long long seed;
    unsigned long long thr_xr;
    IslandState* st;
    double* trace;
    long long pair0;               // first global pair id
};

struct WorkList {
    const uint8_t** ptrs;          // [cap]
    double* obj;                   // [cap]
    double* fit;                   // [cap]
    long long* count;              // device counter
    unsigned long long* total;     // running count of evaluations (optional)
};

// ------------------------------------------------------------------ launchers
struct EvalConfig {
    int G, warps, groups_per_cta, blocks_per_sm;
    int depth;   // K1 pipeline: 2 = two pops in flight, body unrolled 2x; 4 = two in flight, unrolled
                 // 4x (J >= 300); 3 = three in flight, unrolled 6x (J >= 1000)
    GroupLayout gl;
    BucketLayout bl;
    size_t smem;
};
// warps_cap: CTA size cap in warps (0 = 16); the CTA is also capped by shared memory.
int eval_config(const DevInst& I, int sm_count, int warps_cap, EvalConfig* cfg);
cudaError_t launch_eval(const DevInst& I, const EvalConfig& cfg, const EvalItems& W, long long max_items,
                        int sm_count, bool schedule, cudaStream_t st);
// random rows: item i seeded with seed_i = per_item ? derive_seed(base, first + i) : base and
// draw offset off_i = per_item ? 0 : (first + i) * L (random_int_chromosome, chromosome.cpp:68-74)
cudaError_t launch_random_rows(const DevInst& I, uint8_t* out, long long stride, long long n,
                               unsigned long long base, long long first, bool per_item, cudaStream_t st);
cudaError_t launch_pack_bits(const DevInst& I, const uint8_t* rows, long long row_stride,
                             const long long* src_idx, unsigned long long* words, const long long* dst_idx,
                             long long n, bool with_complement, const uint16_t* bit_stage, cudaStream_t st);
cudaError_t launch_unpack_rows(const DevInst& I, const unsigned long long* words, const long long* src_idx,
                               uint8_t* rows, long long row_stride, const long long* dst_idx, long long n,
                               cudaStream_t st);
cudaError_t launch_rows_from_int(const DevInst& I, const int32_t* genes_job_major, const uint8_t* genes_u8,
                                 uint8_t* rows, long long n, cudaStream_t st);
cudaError_t launch_rows_to_int(const DevInst& I, const uint8_t* rows, long long row_stride,
                               const long long* src_idx, int32_t* out, long long n, cudaStream_t st);

// one GA generation over every island of a joint step = launch_breed, launch_eval over the work
// list (n_dev = wl.count), launch_commit
cudaError_t launch_breed(const DevInst& I, const CellIsland* cells_dev, int nc, long long n_cells,
                         const PseudoIsland* pseudo_dev, int np, long long n_pairs, const WorkList& wl,
                         cudaStream_t st);
cudaError_t launch_commit(const DevInst& I, const CellIsland* cells_dev, int nc, const PseudoIsland* pseudo_dev,
                          int np, const WorkList& wl, cudaStream_t st);
// mode 0: refresh best index/fitness; 2: also seed the pseudo archive from every member
cudaError_t launch_island_stats(const DevInst& I, const CellIsland* cells_dev, int nc, const PseudoIsland* pseudo_dev,
                                int np, int mode, cudaStream_t st);

// migration (K5)
size_t sort_temp_bytes(long long n);
cudaError_t launch_sort_desc(const double* fit, long long n, double* keys_tmp, double* keys_out,
                             long long* idx_in, long long* idx_out, void* temp, size_t temp_bytes,
                             cudaStream_t st);
// pk_*: install the k migrants of a packet (rows / words + fit/obj) instead of the source island's
cudaError_t launch_migrate_c2p(const DevInst& I, const CellIsland& c, const PseudoIsland& p,
                               const long long* best_c, const long long* worst_p, int k, int parity,
                               const uint16_t* bit_stage, cudaStream_t st, const uint8_t* pk_rows = nullptr,
                               const double* pk_fo = nullptr);
cudaError_t launch_migrate_p2c(const DevInst& I, const PseudoIsland& p, const CellIsland& c,
                               const long long* best_p, const long long* worst_c, int k, int parity,
                               cudaStream_t st, const unsigned long long* pk_words = nullptr,
                               const double* pk_fo = nullptr);
// migrant packets: [fit[k]][obj[k]][k rows of S*Jpad bytes | k members of W words]
cudaError_t launch_export_cell(const DevInst& I, const CellIsland& c, const long long* best_c, int k, int parity,
                               uint8_t* rows, double* fo, cudaStream_t st);
cudaError_t launch_export_pseudo(const DevInst& I, const PseudoIsland& p, const long long* best_p, int k,
                                 unsigned long long* words, double* fo, cudaStream_t st);
cudaError_t launch_fill_seq(long long* idx, long long n, cudaStream_t st);
// checked build (-DFFSGA_CHECKED): first failed device check, 0 = none; -1 in a normal build
cudaError_t checked_status(long long* status, bool reset);
// compute_cell of one cell on an explicit stream state (cellular.cpp:157-162)
cudaError_t launch_cell_candidate(const DevInst& I, const CellIsland& c, int cell, unsigned long long stream_seed,
                                  int parity, uint8_t* out, unsigned long long* draws, cudaStream_t st);

}  // namespace ffsga_dev
