/*
 * ffsga_oracle.h -- CPU restatement of the reference hot path (TEST INFRASTRUCTURE ONLY).
 *
 * This is the parity checker, not the product.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load it.  The product path
 * (paper_1903_10722_b200, libffsga_cuda.so) never links or calls this code.
 *
 * Every function restates one reference function; the citation is given next to it
 * (paths relative to the reference tree, proj/...).  Parity is pinned two ways
 * (tests/test_oracle_golden.py, tests/test_oracle_vs_ref.py):
 *   1. the golden vectors of the reference's own unit tests (proj/tests/test_*.cpp);
 *   2. the reference itself, compiled from its sources into oracle/_ref/ (oracle/Makefile).
 *
 * Arithmetic contract: plain C doubles, built with -ffp-contract=off exactly like the
 * reference core (proj/src/CMakeLists.txt:16).
 */
#ifndef FFSGA_ORACLE_H
#define FFSGA_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- RNG: proj/include/ffsga/rng.hpp:14-62 ---------------------------------------- */
uint64_t orc_rng_next_u64(uint64_t* state);
double orc_rng_next_unit(uint64_t* state);
double orc_rng_next_uniform(uint64_t* state, double lo, double hi);
int orc_rng_next_index(uint64_t* state, int n);
int orc_rng_next_coin(uint64_t* state, double p);
uint64_t orc_derive_seed(uint64_t base, uint64_t key);

/* ---- Instance: proj/include/ffsga/instance.hpp:12-37 ------------------------------ */
typedef struct {
    int num_jobs;
    int num_stages;
    int* machines_per_stage;  /* S */
    int* stage_offset;        /* S+1 */
    int machines_total;
    double* proc;             /* J * machines_total, [job][stage_offset[s]+m] */
    double* release;          /* J */
    double* due;              /* J */
    double weight;
} orc_instance;

/* Allocates and fills an instance from caller arrays (proc job-major as the reference). */
orc_instance* orc_instance_new(int jobs, int stages, const int* machines, const double* proc,
                               const double* release, const double* due, double weight);
/* proj/src/generator.cpp:11-48 */
orc_instance* orc_generate(int jobs, int stages, const int* machines, double weight,
                           uint64_t seed, int integer_times);
void orc_instance_free(orc_instance* inst);
/* copy-out helpers for tests */
void orc_instance_export(const orc_instance* inst, double* proc, double* release, double* due);

/* proj/src/model.cpp:151-181 */
double orc_mean_job_load(const orc_instance* inst, int job);
double orc_mean_total_load(const orc_instance* inst);
double orc_estimate_emax(const orc_instance* inst);

/* ---- Decoder + evaluator: proj/src/model.cpp:61-149,183-195 ----------------------- */
typedef struct {
    double makespan, total_tardiness, objective, fitness, emax_used;
} orc_report;

/* proj/src/model.cpp:98-105 */
void orc_release_order(const orc_instance* inst, int* order);
/* Evaluator::score (proj/src/model.cpp:192-195).  Returns 0 on success, or -1 and fills
 * bad_job / bad_stage for an out-of-range gene (the ContractError of model.cpp:81-83).
 * When the schedule pointers are non-NULL the full timetable is written ([job][stage]). */
int orc_score(const orc_instance* inst, const int* genes, double emax, orc_report* rep,
              int* sched_machine, double* sched_start, double* sched_completion,
              int* bad_job, int* bad_stage);
/* proj/tests/oracle.cpp:7-45 -- the reference's own independent selection-sort simulator,
 * restated as a second decoder path. */
void orc_simulate_selection(const orc_instance* inst, const int* genes, orc_report* rep);

/* ---- Genome: proj/src/chromosome.cpp:10-74 ---------------------------------------- */
typedef struct {
    int num_jobs, num_stages;
    int bits_per_stage[256];
    int stage_bit_offset[257];
    int bits_per_job, total_bits;
} orc_bit_layout;
int orc_bit_layout_for(const orc_instance* inst, orc_bit_layout* out); /* -1 if S > 256 */
void orc_int_to_bits(const orc_bit_layout* lay, const int* machines, const int* genes,
                     uint8_t* bits);
void orc_bits_to_int(const orc_bit_layout* lay, const int* machines, const uint8_t* bits,
                     int* genes);
void orc_random_int_chromosome(const orc_instance* inst, uint64_t* rng_state, int* genes);

/* ---- Cellular island: proj/src/cellular.cpp:12-195 -------------------------------- */
typedef struct {
    const orc_instance* inst;
    double emax;
    int width, height, size, radius, neighbors_per_cell;
    double crossover_rate, mutation_rate;
    uint64_t island_seed, generation;
    int* genes;        /* size * L, job-major per cell */
    double* fitness;
    double* objective;
    int* slots;        /* size * neighbors_per_cell */
} orc_cellular;

int orc_grid_shape_for(int population, int* width, int* height); /* -1 on ConfigError */
/* proj/src/cellular.cpp:12-27 ; returns neighbor count, writes slot = y*W+x */
int orc_neighborhood_slots(int x, int y, int width, int height, int radius, int* slots);
/* proj/src/cellular.cpp:29-36 */
void orc_sort_island(const double* fitness, int n, int* order);
/* ctor proj/src/cellular.cpp:69-88 (init_genes == NULL) or 90-102 (explicit cells) */
orc_cellular* orc_cellular_new(const orc_instance* inst, double emax, int width, int height,
                               int radius, double crossover_rate, double mutation_rate,
                               uint64_t island_seed, const int* init_genes);
void orc_cellular_free(orc_cellular* g);
/* compute_cell (proj/src/cellular.cpp:116-155) on an explicit stream; child written to
 * child_genes, returns 1 if the child replaces the cell. */
int orc_cellular_candidate(const orc_cellular* g, int index, uint64_t stream_seed,
                           int* child_genes, double* fit, double* obj);
/* same, also returning the number of draws compute_cell consumed */
int orc_cellular_candidate_draws(const orc_cellular* g, int index, uint64_t stream_seed,
                                 int* child_genes, double* fit, double* obj, uint64_t* draws);
void orc_cellular_step(orc_cellular* g); /* proj/src/cellular.cpp:164-182 */
int orc_cellular_best_index(const orc_cellular* g); /* :184-189 */
void orc_cellular_install(orc_cellular* g, int index, const int* genes, double fit, double obj);

/* ---- Pseudo island: proj/src/pseudo.cpp:11-113 ------------------------------------ */
typedef struct {
    const orc_instance* inst;
    double emax;
    orc_bit_layout layout;
    int size;
    double crossover_rate;
    uint64_t island_seed, generation;
    uint8_t* members;  /* size * total_bits, one byte per bit (reference BitChromosome) */
    double* fitness;
    double* objective;
    uint8_t* archive;
    double archive_fitness, archive_objective;
} orc_pseudo;

/* pair_step (proj/src/pseudo.cpp:11-29); returns 1 if the crossover applied */
int orc_pair_step(const uint8_t* a, const uint8_t* b, int nbits, uint64_t* rng_state,
                  double crossover_rate, uint8_t* child1, uint8_t* child2);
orc_pseudo* orc_pseudo_new(const orc_instance* inst, double emax, int population,
                           double crossover_rate, uint64_t island_seed);
void orc_pseudo_free(orc_pseudo* p);
void orc_pseudo_step(orc_pseudo* p);             /* :59-89 */
int orc_pseudo_best_index(const orc_pseudo* p);  /* :91-96 */
void orc_pseudo_install(orc_pseudo* p, int index, const uint8_t* bits, double fit, double obj);

/* ---- Migration: proj/src/migration.cpp:9-69 --------------------------------------- */
double orc_compute_beta(double fit_a, double fit_b);
double orc_compute_alpha(double beta, double theta);
/* direction: 0 none, 1 a_to_b (cellular -> pseudo), 2 b_to_a */
void orc_decide(double fit_a, double fit_b, double theta, int island_population, double* beta,
                double* alpha, int* direction, int* migrants);
void orc_migrate_cellular_to_pseudo(const orc_cellular* from, orc_pseudo* to, int k);
void orc_migrate_pseudo_to_cellular(const orc_pseudo* from, orc_cellular* to, int k);

/* ---- Solver drive(): proj/src/solver.cpp:76-198 ----------------------------------- */
typedef struct {
    int population, generations, migration_gap;
    double theta;
    double cellular_crossover, cellular_mutation;
    int radius;
    double pseudo_crossover;
    int mode; /* 0 dual, 1 cellular only, 2 pseudo only */
    uint64_t seed;
    int grid_w, grid_h; /* 0 = grid_shape_for */
    int pseudo_fit_from_archive;
} orc_run_config;

typedef struct {
    double best_objective, best_fitness, best_makespan, best_tardiness, emax;
    int* best_chromosome;    /* L */
    double* trace_combined;  /* generations */
    double* trace_a;         /* generations or NULL */
    double* trace_b;
    int num_migrations;
    uint64_t* mig_generation;
    double* mig_beta;
    double* mig_alpha;
    int* mig_direction;
    int* mig_migrants;
} orc_run_result;

/* returns 0, or -1 on a configuration error */
int orc_run(const orc_run_config* cfg, const orc_instance* inst, orc_run_result* out);
void orc_run_result_free(orc_run_result* r);

#ifdef __cplusplus
}
#endif
#endif
