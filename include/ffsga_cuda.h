/*
 * ffsga_cuda.h -- C ABI of the B200 (sm_100a) FFS hot path.
 *
 * Plain C types only (pointers, sizes, status codes): this is the boundary a reference-side
 * binding (pybind11 / ctypes / cgo ...) would call.  Every entry point cites the reference
 * interface it replaces (paths relative to the reference tree, proj/...).  INTEGRATION.md shows
 * the reference-side bindings.
 *
 * Conventions
 *   - every function returns an ffsga_status; on failure ffsga_cuda_last_error() returns the
 *     message of the failing call on this thread (thread-local).  Status mapping mirrors the
 *     reference exception hierarchy (proj/include/ffsga/errors.hpp:9-31):
 *       FFSGA_ERR_CONTRACT <- ContractError, FFSGA_ERR_CONFIG <- ConfigError.
 *   - chromosomes cross the boundary job-major (gene i = machine of job i/S at stage i%S,
 *     proj/include/ffsga/chromosome.hpp:12-16); bit chromosomes one byte per bit, exactly the
 *     reference BitChromosome (chromosome.hpp:37-40).
 *   - host pointers unless the name says _device.  Calls are synchronous unless they say async.
 *   - handles are thread-safe per handle; islands stepped together must share one instance.
 *   - there is no CPU fallback: without a usable sm_100 device every call fails with
 *     FFSGA_ERR_CUDA.
 */
#ifndef FFSGA_CUDA_H
#define FFSGA_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FFSGA_CUDA_ABI_VERSION 1

typedef enum {
    FFSGA_OK = 0,
    FFSGA_ERR_CONTRACT = 1, /* ContractError: precondition violated (bad gene, size, index) */
    FFSGA_ERR_CONFIG = 2,   /* ConfigError: invalid island / run configuration */
    FFSGA_ERR_CUDA = 3,     /* CUDA runtime failure or no sm_100 device */
    FFSGA_ERR_OOM = 4,      /* device allocation failed */
    FFSGA_ERR_ARG = 5       /* null handle / pointer */
} ffsga_status;

typedef struct ffsga_cuda_instance_t* ffsga_cuda_instance;
typedef struct ffsga_cuda_batch_t* ffsga_cuda_batch;
typedef struct ffsga_cuda_cellular_t* ffsga_cuda_cellular;
typedef struct ffsga_cuda_pseudo_t* ffsga_cuda_pseudo;

const char* ffsga_cuda_last_error(void);
int ffsga_cuda_abi_version(void);
int ffsga_cuda_device_count(int* count);

/* ---- instance ---------------------------------------------------------------------------
 * Replaces: ffsga::Instance (proj/include/ffsga/instance.hpp:12-37) as seen by
 * Evaluator(const Instance&, double emax) (proj/include/ffsga/model.hpp:57-70).  proc is the
 * reference's flat [job][stage_offset[s] + m] array (instance.hpp:25-27).  emax is the fitness
 * bound every evaluation on this handle uses (estimate_emax, model.cpp:167-181, is host-side).
 * Config errors: machines_per_stage outside [1, 32], num_jobs > 65000, or a processing time
 * below the ulp of the schedule horizon (the merge-ordered decoder needs strictly increasing
 * completions per machine). */
int ffsga_cuda_instance_create(int device, int num_jobs, int num_stages, const int32_t* machines_per_stage,
                               const double* proc, const double* release, const double* due,
                               double weight, double emax, ffsga_cuda_instance* out);
int ffsga_cuda_instance_destroy(ffsga_cuda_instance inst);
/* row_stride = Jpad (bytes per device gene row); group_lanes = decoder lanes per chromosome;
 * total_bits = BitLayout::total_bits (chromosome.cpp:10-26) */
int ffsga_cuda_instance_info(ffsga_cuda_instance inst, int* row_stride, int* group_lanes, int* total_bits,
                             int* smem_per_group);

/* ---- K1: batch evaluation ------------------------------------------------------------------
 * Replaces: ObjectiveReport Evaluator::score(std::span<const int>) (model.hpp:61,
 * model.cpp:192-195) applied to n chromosomes.  genes: n * J*S job-major int32.  Outputs are
 * n doubles each; makespan / tardiness may be NULL.  An out-of-range gene makes the call fail
 * with FFSGA_ERR_CONTRACT and the reference message of the first offending chromosome
 * ("decode: machine index out of range at job J stage S", model.cpp:81-83).
 * A genes buffer in page-locked host memory (cudaHostAlloc / cudaHostRegister) is read in place
 * by the copy engine; pageable buffers go through the library's pinned staging pair. */
int ffsga_cuda_evaluate(ffsga_cuda_instance inst, const int32_t* genes, int64_t n, double* objective,
                        double* fitness, double* makespan, double* tardiness);
/* Same with one byte per gene (the compact host layout of the e2e decoder benchmark). */
int ffsga_cuda_evaluate_u8(ffsga_cuda_instance inst, const uint8_t* genes, int64_t n, double* objective,
                           double* fitness, double* makespan, double* tardiness);
/* Same for a population already resident in device memory (torch / DLPack
 * tensors): genes, objective, fitness (and the optional makespan / tardiness) are DEVICE pointers
 * of the instance's device, genes job-major one byte per gene.  The work is ordered after
 * everything already queued on `stream` (a cudaStream_t; NULL = legacy default stream) and
 * everything queued on it afterwards sees the results.  Out-of-range genes fail as above. */
int ffsga_cuda_evaluate_device(ffsga_cuda_instance inst, const uint8_t* genes, int64_t n, double* objective,
                               double* fitness, double* makespan, double* tardiness, void* stream);

/* ---- K7: schedule materialization ----------------------------------------------------------
 * Replaces: Schedule decode(const Instance&, span<const int>) (model.hpp:42, model.cpp:124-139)
 * followed by evaluate(...) (model.cpp:141-149).  machine/start/completion: J*S job-major.
 * report5 (optional) = {makespan, total_tardiness, objective, fitness, emax_used}. */
int ffsga_cuda_decode(ffsga_cuda_instance inst, const int32_t* genes, int32_t* machine, double* start,
                      double* completion, double* report5);

/* ---- device-resident batches (decoder sweep) -------------------------------- */
int ffsga_cuda_batch_create(ffsga_cuda_instance inst, int64_t capacity, ffsga_cuda_batch* out);
int ffsga_cuda_batch_destroy(ffsga_cuda_batch b);
/* K2: chromosome i = random_int_chromosome(inst, Rng(derive_seed(base_seed, first + i)))
 * (chromosome.cpp:68-74, rng.hpp:55-58); async */
int ffsga_cuda_batch_fill_random(ffsga_cuda_batch b, uint64_t base_seed, int64_t first, int64_t n);
/* host job-major genes -> device rows (int32 or one byte per gene); async after staging */
int ffsga_cuda_batch_upload(ffsga_cuda_batch b, const int32_t* genes, int64_t n);
int ffsga_cuda_batch_upload_u8(ffsga_cuda_batch b, const uint8_t* genes, int64_t n);
/* K1 over the first n rows; async */
int ffsga_cuda_batch_evaluate(ffsga_cuda_batch b, int64_t n);
/* synchronous D2H of results (any pointer may be NULL); also reports a pending gene error */
int ffsga_cuda_batch_results(ffsga_cuda_batch b, int64_t n, double* objective, double* fitness,
                             double* makespan, double* tardiness);
/* device pointers of the result arrays (objective, fitness), for zero-copy consumers */
int ffsga_cuda_batch_device_results(ffsga_cuda_batch b, const double** objective, const double** fitness);
/* job-major int32 copy of rows [first, first+n) */
int ffsga_cuda_batch_download(ffsga_cuda_batch b, int64_t first, int64_t n, int32_t* genes);
int ffsga_cuda_batch_sync(ffsga_cuda_batch b);
/* milliseconds of the last batch_evaluate kernel (CUDA events on the launching stream) */
int ffsga_cuda_batch_last_eval_ms(ffsga_cuda_batch b, float* ms);

/* ---- cellular island -------------------------------------------------------------------------
 * Replaces: ffsga::CellGrid (proj/include/ffsga/cellular.hpp:47-115, cellular.cpp:50-195).
 * init_genes == NULL: population from one sequential Rng(island_seed) stream (cellular.cpp:84-86);
 * otherwise width*height explicit job-major chromosomes (cellular.cpp:90-102). */
int ffsga_cuda_cellular_create(ffsga_cuda_instance inst, int width, int height, int radius,
                               double crossover_rate, double mutation_rate, uint64_t island_seed,
                               const int32_t* init_genes, ffsga_cuda_cellular* out);
int ffsga_cuda_cellular_destroy(ffsga_cuda_cellular c);
int ffsga_cuda_cellular_size(ffsga_cuda_cellular c, int* size, int* width, int* height, int* neighbors);
int ffsga_cuda_cellular_generation(ffsga_cuda_cellular c, uint64_t* generation);
/* fitness()/objective() spans (cellular.hpp:81-82) */
int ffsga_cuda_cellular_read(ffsga_cuda_cellular c, double* fitness, double* objective);
/* cell(i) (cellular.hpp:83); index < 0 copies the whole population (size * J*S) */
int ffsga_cuda_cellular_genes(ffsga_cuda_cellular c, int index, int32_t* genes);
/* neighbor_slots(i) (cellular.hpp:68-71) */
int ffsga_cuda_cellular_slots(ffsga_cuda_cellular c, int index, int32_t* slots);
/* best_index / best_fitness / best_objective (cellular.cpp:184-189) */
int ffsga_cuda_cellular_best(ffsga_cuda_cellular c, int* index, double* fitness, double* objective);
/* cell_candidate (cellular.cpp:157-162): compute_cell of `index` against the current state on
 * the stream whose state is `stream_state` (the state of an ffsga::Rng).  Returns the candidate
 * (child if replaced, else the current cell) and how many draws the reference consumes, so the
 * caller can advance its Rng. */
int ffsga_cuda_cellular_candidate(ffsga_cuda_cellular c, int index, uint64_t stream_state, int32_t* genes,
                                  double* fitness, double* objective, int* replaced, uint64_t* draws_used);
/* install (cellular.cpp:191-195) */
int ffsga_cuda_cellular_install(ffsga_cuda_cellular c, int index, const int32_t* genes, double fitness,
                                double objective);

/* ---- pseudo island ----------------------------------------------------------------------------
 * Replaces: ffsga::PairPopulation (proj/include/ffsga/pseudo.hpp:35-81, pseudo.cpp:31-113). */
int ffsga_cuda_pseudo_create(ffsga_cuda_instance inst, int population, double crossover_rate,
                             uint64_t island_seed, ffsga_cuda_pseudo* out);
int ffsga_cuda_pseudo_destroy(ffsga_cuda_pseudo p);
int ffsga_cuda_pseudo_size(ffsga_cuda_pseudo p, int* size, int* total_bits);
int ffsga_cuda_pseudo_generation(ffsga_cuda_pseudo p, uint64_t* generation);
int ffsga_cuda_pseudo_read(ffsga_cuda_pseudo p, double* fitness, double* objective);
/* member(i) as one byte per bit; index < 0 copies all members (size * total_bits) */
int ffsga_cuda_pseudo_member(ffsga_cuda_pseudo p, int index, uint8_t* bits);
int ffsga_cuda_pseudo_best(ffsga_cuda_pseudo p, int* index, double* fitness, double* objective);
/* archive_chromosome / archive_fitness / archive_objective (pseudo.hpp:58-60); bits may be NULL */
int ffsga_cuda_pseudo_archive(ffsga_cuda_pseudo p, double* fitness, double* objective, uint8_t* bits);
/* bits_to_int(archive_chromosome()) as job-major int32 genes (solver.cpp:182) */
int ffsga_cuda_pseudo_archive_genes(ffsga_cuda_pseudo p, int32_t* genes);
/* install (pseudo.cpp:98-104): the archive absorbs the installed score */
int ffsga_cuda_pseudo_install(ffsga_cuda_pseudo p, int index, const uint8_t* bits, double fitness,
                              double objective);

/* ---- the generation loop ----------------------------------------------------------------------
 * Replaces: CellGrid::step (cellular.cpp:164-182) and PairPopulation::step (pseudo.cpp:59-89),
 * `generations` times, for every listed island jointly (one fused launch sequence per
 * generation, the B200 form of the concurrent island segment of solver.cpp:126-139).
 * trace_cellular[i*generations + g] = best_objective() of cellular island i after generation g
 * (solver.cpp:113); trace_pseudo[...] = archive_objective() (solver.cpp:121).  Either may be NULL.
 * The reference's `workers` argument has no device meaning: results never depend on it. */
int ffsga_cuda_step(const ffsga_cuda_cellular* cells, int n_cells, const ffsga_cuda_pseudo* pseudos,
                    int n_pseudos, int generations, double* trace_cellular, double* trace_pseudo);

/* ---- migration (K5) -------------------------------------------------------------------------
 * Replaces: migrate_cellular_to_pseudo / migrate_pseudo_to_cellular (migration.hpp:45-46,
 * migration.cpp:47-69).  k best of the source (sort_island order, cellular.cpp:29-36) overwrite
 * the k worst of the destination.  The policy (decide, migration.cpp:21-36) is host-side. */
int ffsga_cuda_migrate_cellular_to_pseudo(ffsga_cuda_cellular from, ffsga_cuda_pseudo to, int k);
int ffsga_cuda_migrate_pseudo_to_cellular(ffsga_cuda_pseudo from, ffsga_cuda_cellular to, int k);

/* Cross-device migration halves (the same transfer as above, split at the wire so the rows can
 * travel between GPUs): export the k best of one island in sort_island order, import them over
 * the k worst of the other (best lands on worst).  Cellular islands export job-major int32
 * genes and import bit chromosomes (bits_to_int on the device); pseudo islands export bit
 * chromosomes (one byte per bit) and import int32 genes (int_to_bits on the device). */
int ffsga_cuda_cellular_export(ffsga_cuda_cellular c, int k, int32_t* genes, double* fitness, double* objective);
int ffsga_cuda_pseudo_export(ffsga_cuda_pseudo p, int k, uint8_t* bits, double* fitness, double* objective);
int ffsga_cuda_cellular_import(ffsga_cuda_cellular c, int k, const uint8_t* bits, const double* fitness,
                               const double* objective);
int ffsga_cuda_pseudo_import(ffsga_cuda_pseudo p, int k, const int32_t* genes, const double* fitness,
                             const double* objective);

/* Device-resident halves (the data plane between GPUs: the packet is device memory that NCCL or
 * a peer copy moves over NVLink; nothing is staged through the host).  A migrant packet is
 * [fitness[k] f64][objective[k] f64][payload]: payload = k stage-major gene rows (from a
 * cellular island) or k packed bit chromosomes of ceil(total_bits/64) u64 words, LSB-first
 * (from a pseudo island).  Export and import are ordered on `stream` (a cudaStream_t; NULL =
 * the legacy default stream) and never synchronise the host.  A cellular island imports a
 * pseudo island's packet and vice versa; best lands on worst, and a pseudo import feeds the
 * archive in install order (migration.cpp:47-69, pseudo.cpp:98-113). */
int ffsga_cuda_packet_bytes(ffsga_cuda_instance inst, int from_kind /* 0 cellular, 1 pseudo */, int k,
                            int64_t* bytes);
int ffsga_cuda_cellular_export_device(ffsga_cuda_cellular c, int k, void* packet, void* stream);
int ffsga_cuda_pseudo_export_device(ffsga_cuda_pseudo p, int k, void* packet, void* stream);
int ffsga_cuda_cellular_import_device(ffsga_cuda_cellular c, int k, const void* packet, void* stream);
int ffsga_cuda_pseudo_import_device(ffsga_cuda_pseudo p, int k, const void* packet, void* stream);
/* island statistics into device memory, ordered on `stream`: out4 = {best fitness, best
 * objective, archive fitness, archive objective} (best_index of cellular.cpp:184-189 /
 * pseudo.cpp:91-96; archive of pseudo.hpp:78-80, -1 / 0 for a cellular island) -- what the
 * rendezvous policy (solver.cpp:142-163) and the champion rule (solver.cpp:175-183) read */
int ffsga_cuda_cellular_state_device(ffsga_cuda_cellular c, double* out4, void* stream);
int ffsga_cuda_pseudo_state_device(ffsga_cuda_pseudo p, double* out4, void* stream);

/* ---- measurement ------------------------------------------------------------------------------
 * Per-kernel CUDA-event timing on the launching stream (off by default).  When enabled, every
 * k_eval launch of a batch or of ffsga_cuda_step is bracketed by events; totals accumulate. */
int ffsga_cuda_set_timing(ffsga_cuda_instance inst, int enabled);
/* total milliseconds and launch count of: 0 = K1 eval, 1 = K3+K4 breed, 2 = K6 commit */
int ffsga_cuda_timing(ffsga_cuda_instance inst, int which, double* ms, int64_t* launches);
/* milliseconds during which at least one launch of that kind was running: the union of the
 * event intervals, so the concurrent cellular and pseudo chains of a joint step count once */
int ffsga_cuda_timing_busy(ffsga_cuda_instance inst, int which, double* busy_ms);
int ffsga_cuda_reset_timing(ffsga_cuda_instance inst);
/* makespan evaluations performed by ffsga_cuda_step on this instance since creation
 * (cellular children + crossed pseudo members; device counter) */
int ffsga_cuda_evaluations(ffsga_cuda_instance inst, int64_t* count);
/* device milliseconds of the last ffsga_cuda_step launch sequence (events on its stream) */
int ffsga_cuda_last_step_ms(ffsga_cuda_instance inst, float* ms);
/* Diagnostics of a checked build (python build.py --checked -> paper_1903_10722_b200/checked/):
 * the first device-side bounds / invariant check that failed since the last reset, encoded
 * code << 48 | a << 24 | b, 0 when none failed; -1 from a normal build.  Synchronises the
 * device. */
int ffsga_cuda_checked_status(int reset, int64_t* status);
/* kernels launched by this library since load (all kinds) */
int ffsga_cuda_launch_count(int64_t* count);

#ifdef __cplusplus
}
#endif
#endif
