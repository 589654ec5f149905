/*
 * ffsga_oracle.c -- CPU restatement of the reference hot path.  TEST INFRASTRUCTURE ONLY:
 * the checker for the CUDA product, never linked into it.  See ffsga_oracle.h for the
 * contract and the pinning strategy.  Build: oracle/Makefile (-O2 -ffp-contract=off).
 */
#include "ffsga_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9E3779B97F4A7C15ULL

/* std::max / std::min semantics (return the first argument unless the second is larger /
 * smaller), which matters for signed zeros. */
static inline double std_max(double a, double b) { return (a < b) ? b : a; }
static inline double std_min(double a, double b) { return (b < a) ? b : a; }

/* ---------------------------------------------------------------- RNG (rng.hpp:14-62) */
uint64_t orc_rng_next_u64(uint64_t* state) { /* rng.hpp:18-23 */
    uint64_t z = (*state += GAMMA);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ULL;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBULL;
    return z ^ (z >> 31);
}

double orc_rng_next_unit(uint64_t* state) { /* rng.hpp:26-28 */
    return (double)(orc_rng_next_u64(state) >> 11) * 0x1.0p-53;
}

double orc_rng_next_uniform(uint64_t* state, double lo, double hi) { /* rng.hpp:31-36 */
    double v = lo + orc_rng_next_unit(state) * (hi - lo);
    if (v >= hi) v = nextafter(hi, lo);
    return v;
}

int orc_rng_next_index(uint64_t* state, int n) { /* rng.hpp:39-43 */
    int v = (int)(orc_rng_next_unit(state) * (double)n);
    return v < n ? v : n - 1;
}

int orc_rng_next_coin(uint64_t* state, double p) { /* rng.hpp:45 */
    return orc_rng_next_unit(state) < p;
}

uint64_t orc_derive_seed(uint64_t base, uint64_t key) { /* rng.hpp:55-58 */
    uint64_t s = base + key * GAMMA;
    return orc_rng_next_u64(&s);
}

/* ------------------------------------------------------------ Instance (model.cpp:11-16) */
static orc_instance* alloc_instance(int jobs, int stages, const int* machines) {
    orc_instance* inst = (orc_instance*)calloc(1, sizeof(orc_instance));
    inst->num_jobs = jobs;
    inst->num_stages = stages;
    inst->machines_per_stage = (int*)malloc(sizeof(int) * stages);
    inst->stage_offset = (int*)malloc(sizeof(int) * (stages + 1));
    inst->stage_offset[0] = 0;
    for (int s = 0; s < stages; ++s) {
        inst->machines_per_stage[s] = machines[s];
        inst->stage_offset[s + 1] = inst->stage_offset[s] + machines[s];
    }
    inst->machines_total = inst->stage_offset[stages];
    inst->proc = (double*)calloc((size_t)jobs * inst->machines_total, sizeof(double));
    inst->release = (double*)calloc(jobs, sizeof(double));
    inst->due = (double*)calloc(jobs, sizeof(double));
    return inst;
}

orc_instance* orc_instance_new(int jobs, int stages, const int* machines, const double* proc,
                               const double* release, const double* due, double weight) {
    orc_instance* inst = alloc_instance(jobs, stages, machines);
    memcpy(inst->proc, proc, sizeof(double) * (size_t)jobs * inst->machines_total);
    memcpy(inst->release, release, sizeof(double) * jobs);
    memcpy(inst->due, due, sizeof(double) * jobs);
    inst->weight = weight;
    return inst;
}

void orc_instance_free(orc_instance* inst) {
    if (!inst) return;
    free(inst->machines_per_stage);
    free(inst->stage_offset);
    free(inst->proc);
    free(inst->release);
    free(inst->due);
    free(inst);
}

void orc_instance_export(const orc_instance* inst, double* proc, double* release, double* due) {
    if (proc) memcpy(proc, inst->proc, sizeof(double) * (size_t)inst->num_jobs * inst->machines_total);
    if (release) memcpy(release, inst->release, sizeof(double) * inst->num_jobs);
    if (due) memcpy(due, inst->due, sizeof(double) * inst->num_jobs);
}

static inline double proc_time(const orc_instance* inst, int j, int s, int m) {
    return inst->proc[(size_t)j * inst->machines_total + inst->stage_offset[s] + m];
}

double orc_mean_job_load(const orc_instance* inst, int job) { /* model.cpp:151-159 */
    double total = 0.0;
    for (int s = 0; s < inst->num_stages; ++s) {
        double sum = 0.0;
        for (int m = 0; m < inst->machines_per_stage[s]; ++m) sum += proc_time(inst, job, s, m);
        total += sum / inst->machines_per_stage[s];
    }
    return total;
}

double orc_mean_total_load(const orc_instance* inst) { /* model.cpp:161-165 */
    double total = 0.0;
    for (int j = 0; j < inst->num_jobs; ++j) total += orc_mean_job_load(inst, j);
    return total;
}

double orc_estimate_emax(const orc_instance* inst) { /* model.cpp:167-181 */
    double horizon = 0.0;
    for (int j = 0; j < inst->num_jobs; ++j) horizon = std_max(horizon, inst->release[j]);
    for (int j = 0; j < inst->num_jobs; ++j)
        for (int s = 0; s < inst->num_stages; ++s) {
            double worst = 0.0;
            for (int m = 0; m < inst->machines_per_stage[s]; ++m)
                worst = std_max(worst, proc_time(inst, j, s, m));
            horizon += worst;
        }
    double tardiness_bound = 0.0;
    for (int j = 0; j < inst->num_jobs; ++j)
        tardiness_bound += std_max(0.0, horizon - inst->due[j]);
    return inst->weight * tardiness_bound + horizon;
}

orc_instance* orc_generate(int jobs, int stages, const int* machines, double weight,
                           uint64_t seed, int integer_times) { /* generator.cpp:11-48 */
    orc_instance* inst = alloc_instance(jobs, stages, machines);
    inst->weight = weight;
    uint64_t rng = seed;
    for (int j = 0; j < jobs; ++j)
        for (int s = 0; s < stages; ++s)
            for (int m = 0; m < machines[s]; ++m) {
                double p = orc_rng_next_uniform(&rng, 1.0, 5.0);
                if (integer_times) p = round(p);
                inst->proc[(size_t)j * inst->machines_total + inst->stage_offset[s] + m] = p;
            }
    double total_load = orc_mean_total_load(inst);
    for (int j = 0; j < jobs; ++j) inst->release[j] = orc_rng_next_uniform(&rng, 0.0, total_load);
    for (int j = 0; j < jobs; ++j) {
        double slack = orc_rng_next_uniform(&rng, 0.0, 2.0);
        inst->due[j] = inst->release[j] + orc_mean_job_load(inst, j) * (1.0 + slack);
    }
    return inst;
}

/* ------------------------------------------------------- Decoder (model.cpp:61-149) */
/* Merge sort of job indices by (key[j], j); any correct sort yields the same permutation
 * because the order is total (model.cpp:73-75, 101-103). */
static void sort_by_key(int* idx, int* tmp, int n, const double* key) {
    if (n < 2) return;
    int h = n / 2;
    sort_by_key(idx, tmp, h, key);
    sort_by_key(idx + h, tmp, n - h, key);
    int a = 0, b = h, o = 0;
    while (a < h && b < n) {
        int x = idx[a], y = idx[b];
        int y_first = key[y] < key[x] || (key[y] == key[x] && y < x);
        tmp[o++] = y_first ? idx[b++] : idx[a++];
    }
    while (a < h) tmp[o++] = idx[a++];
    while (b < n) tmp[o++] = idx[b++];
    memcpy(idx, tmp, sizeof(int) * n);
}

void orc_release_order(const orc_instance* inst, int* order) { /* model.cpp:98-105 */
    int* tmp = (int*)malloc(sizeof(int) * inst->num_jobs);
    for (int j = 0; j < inst->num_jobs; ++j) order[j] = j;
    sort_by_key(order, tmp, inst->num_jobs, inst->release);
    free(tmp);
}

int orc_score(const orc_instance* inst, const int* genes, double emax, orc_report* rep,
              int* sched_machine, double* sched_start, double* sched_completion, int* bad_job,
              int* bad_stage) {
    const int J = inst->num_jobs, S = inst->num_stages;
    int* order = (int*)malloc(sizeof(int) * J);
    int* tmp = (int*)malloc(sizeof(int) * J);
    double* ready = (double*)malloc(sizeof(double) * J);
    int maxm = 1;
    for (int s = 0; s < S; ++s) if (inst->machines_per_stage[s] > maxm) maxm = inst->machines_per_stage[s];
    double* avail = (double*)malloc(sizeof(double) * maxm);
    int status = 0;
    /* run_list_schedule, model.cpp:61-96 */
    for (int j = 0; j < J; ++j) ready[j] = inst->release[j];
    for (int s = 0; s < S && status == 0; ++s) {
        if (s == 0) {
            orc_release_order(inst, order);
        } else {
            for (int j = 0; j < J; ++j) order[j] = j;
            sort_by_key(order, tmp, J, ready);
        }
        const int machines = inst->machines_per_stage[s];
        for (int m = 0; m < machines; ++m) avail[m] = 0.0;
        for (int k = 0; k < J; ++k) {
            int j = order[k];
            int m = genes[j * S + s];
            if (m < 0 || m >= machines) {
                if (bad_job) *bad_job = j;
                if (bad_stage) *bad_stage = s;
                status = -1;
                break;
            }
            double start = std_max(ready[j], avail[m]);
            double completion = start + proc_time(inst, j, s, m);
            avail[m] = completion;
            ready[j] = completion;
            if (sched_machine) sched_machine[j * S + s] = m;
            if (sched_start) sched_start[j * S + s] = start;
            if (sched_completion) sched_completion[j * S + s] = completion;
        }
    }
    if (status == 0 && rep) { /* report_from_completions, model.cpp:107-120 */
        rep->emax_used = emax;
        rep->makespan = 0.0;
        rep->total_tardiness = 0.0;
        for (int j = 0; j < J; ++j) {
            double c = ready[j];
            rep->makespan = std_max(rep->makespan, c);
            rep->total_tardiness += std_max(0.0, c - inst->due[j]);
        }
        rep->objective = inst->weight * rep->total_tardiness + rep->makespan;
        rep->fitness = std_max(emax - rep->objective, 0.0);
    }
    free(order); free(tmp); free(ready); free(avail);
    return status;
}

void orc_simulate_selection(const orc_instance* inst, const int* genes, orc_report* rep) {
    /* proj/tests/oracle.cpp:7-45: repeated minimum extraction, lowest job on ties */
    const int J = inst->num_jobs, S = inst->num_stages;
    double* entry = (double*)malloc(sizeof(double) * J);
    double* ready = (double*)malloc(sizeof(double) * J);
    double* done = (double*)calloc(J, sizeof(double));
    char* dispatched = (char*)malloc(J);
    double* mfree = (double*)malloc(sizeof(double) * inst->machines_total);
    for (int j = 0; j < J; ++j) entry[j] = ready[j] = inst->release[j];
    for (int i = 0; i < inst->machines_total; ++i) mfree[i] = 0.0;
    for (int s = 0; s < S; ++s) {
        memset(dispatched, 0, J);
        for (int round_ = 0; round_ < J; ++round_) {
            int pick = -1;
            for (int j = 0; j < J; ++j) {
                if (dispatched[j]) continue;
                if (pick == -1 || entry[j] < entry[pick]) pick = j;
            }
            dispatched[pick] = 1;
            int machine = genes[pick * S + s];
            double* slot = &mfree[inst->stage_offset[s] + machine];
            double start = std_max(ready[pick], *slot);
            double finish = start + proc_time(inst, pick, s, machine);
            *slot = finish;
            done[pick] = finish;
        }
        memcpy(entry, done, sizeof(double) * J);
        memcpy(ready, done, sizeof(double) * J);
    }
    rep->makespan = 0.0;
    rep->total_tardiness = 0.0;
    for (int j = 0; j < J; ++j) {
        rep->makespan = std_max(rep->makespan, done[j]);
        rep->total_tardiness += std_max(0.0, done[j] - inst->due[j]);
    }
    rep->objective = inst->weight * rep->total_tardiness + rep->makespan;
    rep->fitness = 0.0;
    rep->emax_used = 0.0;
    free(entry); free(ready); free(done); free(dispatched); free(mfree);
}

/* ------------------------------------------------------ Genome (chromosome.cpp:10-74) */
static int bit_width_u(unsigned v) {
    int w = 0;
    while (v) { ++w; v >>= 1; }
    return w;
}

int orc_bit_layout_for(const orc_instance* inst, orc_bit_layout* out) { /* :10-26 */
    if (inst->num_stages > 256) return -1;
    memset(out, 0, sizeof(*out));
    out->num_jobs = inst->num_jobs;
    out->num_stages = inst->num_stages;
    out->stage_bit_offset[0] = 0;
    for (int s = 0; s < inst->num_stages; ++s) {
        unsigned m = (unsigned)inst->machines_per_stage[s];
        int bits = bit_width_u(m - 1u);
        if (bits < 1) bits = 1;
        out->bits_per_stage[s] = bits;
        out->stage_bit_offset[s + 1] = out->stage_bit_offset[s] + bits;
    }
    out->bits_per_job = out->stage_bit_offset[inst->num_stages];
    out->total_bits = out->num_jobs * out->bits_per_job;
    return 0;
}

static inline int gene_offset(const orc_bit_layout* lay, int gene) {
    return (gene / lay->num_stages) * lay->bits_per_job + lay->stage_bit_offset[gene % lay->num_stages];
}

void orc_int_to_bits(const orc_bit_layout* lay, const int* machines, const int* genes,
                     uint8_t* bits) { /* chromosome.cpp:28-42 */
    (void)machines;
    memset(bits, 0, lay->total_bits);
    const int L = lay->num_jobs * lay->num_stages;
    for (int i = 0; i < L; ++i) {
        int stage = i % lay->num_stages;
        int nb = lay->bits_per_stage[stage];
        int off = gene_offset(lay, i);
        unsigned value = (unsigned)genes[i];
        for (int b = 0; b < nb; ++b) bits[off + b] = (uint8_t)((value >> (nb - 1 - b)) & 1u);
    }
}

void orc_bits_to_int(const orc_bit_layout* lay, const int* machines, const uint8_t* bits,
                     int* genes) { /* chromosome.cpp:44-59 */
    const int L = lay->num_jobs * lay->num_stages;
    for (int i = 0; i < L; ++i) {
        int stage = i % lay->num_stages;
        int nb = lay->bits_per_stage[stage];
        int off = gene_offset(lay, i);
        unsigned value = 0;
        for (int b = 0; b < nb; ++b) value = (value << 1) | bits[off + b];
        genes[i] = (int)(value % (unsigned)machines[stage]);
    }
}

void orc_random_int_chromosome(const orc_instance* inst, uint64_t* rng, int* genes) {
    /* chromosome.cpp:68-74 */
    const int L = inst->num_jobs * inst->num_stages;
    for (int i = 0; i < L; ++i) genes[i] = orc_rng_next_index(rng, inst->machines_per_stage[i % inst->num_stages]);
}

/* ------------------------------------------------ Cellular island (cellular.cpp:12-195) */
int orc_grid_shape_for(int population, int* width, int* height) { /* :38-48 */
    if (population < 4) return -1;
    int best = 1;
    for (int d = 1; d * d <= population; ++d)
        if (population % d == 0) best = d;
    if (best < 2) return -1;
    *width = population / best;
    *height = best;
    return 0;
}

int orc_neighborhood_slots(int x, int y, int width, int height, int radius, int* slots) {
    /* :12-27, flattened as in finish_setup :59-66 */
    int n = 0;
    for (int dy = -radius; dy <= radius; ++dy) {
        int budget = radius - abs(dy);
        for (int dx = -budget; dx <= budget; ++dx) {
            if (dx == 0 && dy == 0) continue;
            int nx = ((x + dx) % width + width) % width;
            int ny = ((y + dy) % height + height) % height;
            if (slots) slots[n] = ny * width + nx;
            ++n;
        }
    }
    return n;
}

void orc_sort_island(const double* fitness, int n, int* order) { /* :29-36 */
    /* fitness descending, index ascending: sort by key = -fitness with index ties */
    double* key = (double*)malloc(sizeof(double) * (n > 0 ? n : 1));
    int* tmp = (int*)malloc(sizeof(int) * (n > 0 ? n : 1));
    for (int i = 0; i < n; ++i) { key[i] = -fitness[i]; order[i] = i; }
    sort_by_key(order, tmp, n, key);
    free(key); free(tmp);
}

orc_cellular* orc_cellular_new(const orc_instance* inst, double emax, int width, int height,
                               int radius, double crossover_rate, double mutation_rate,
                               uint64_t island_seed, const int* init_genes) {
    orc_cellular* g = (orc_cellular*)calloc(1, sizeof(orc_cellular));
    const int L = inst->num_jobs * inst->num_stages;
    g->inst = inst;
    g->emax = emax;
    g->width = width;
    g->height = height;
    g->size = width * height;
    g->radius = radius;
    g->crossover_rate = crossover_rate;
    g->mutation_rate = mutation_rate;
    g->island_seed = island_seed;
    g->genes = (int*)malloc(sizeof(int) * (size_t)g->size * L);
    g->fitness = (double*)malloc(sizeof(double) * g->size);
    g->objective = (double*)malloc(sizeof(double) * g->size);
    if (init_genes) { /* :90-102 */
        memcpy(g->genes, init_genes, sizeof(int) * (size_t)g->size * L);
    } else { /* :84-86, one sequential stream for all cells */
        uint64_t rng = island_seed;
        for (int i = 0; i < g->size; ++i) orc_random_int_chromosome(inst, &rng, g->genes + (size_t)i * L);
    }
    /* finish_setup :50-67 */
    for (int i = 0; i < g->size; ++i) {
        orc_report rep;
        orc_score(inst, g->genes + (size_t)i * L, emax, &rep, NULL, NULL, NULL, NULL, NULL);
        g->fitness[i] = rep.fitness;
        g->objective[i] = rep.objective;
    }
    g->neighbors_per_cell = orc_neighborhood_slots(0, 0, width, height, radius, NULL);
    g->slots = (int*)malloc(sizeof(int) * (size_t)g->size * g->neighbors_per_cell);
    for (int i = 0; i < g->size; ++i)
        orc_neighborhood_slots(i % width, i / width, width, height, radius,
                               g->slots + (size_t)i * g->neighbors_per_cell);
    return g;
}

void orc_cellular_free(orc_cellular* g) {
    if (!g) return;
    free(g->genes); free(g->fitness); free(g->objective); free(g->slots); free(g);
}

static int tournament(const int* slots, int n, const double* fitness, uint64_t* rng) {
    /* cellular.cpp:108-112 */
    int a = slots[orc_rng_next_index(rng, n)];
    int b = slots[orc_rng_next_index(rng, n)];
    return fitness[b] > fitness[a] ? b : a;
}

int orc_cellular_candidate(const orc_cellular* g, int index, uint64_t stream_seed,
                           int* child, double* fit, double* obj) {
    return orc_cellular_candidate_draws(g, index, stream_seed, child, fit, obj, NULL);
}

int orc_cellular_candidate_draws(const orc_cellular* g, int index, uint64_t stream_seed,
                                 int* child, double* fit, double* obj, uint64_t* draws) { /* :116-155 */
    const orc_instance* inst = g->inst;
    const int L = inst->num_jobs * inst->num_stages;
    const int n = g->neighbors_per_cell;
    const int* slots = g->slots + (size_t)index * n;
    uint64_t rng = stream_seed;
    int parent1 = tournament(slots, n, g->fitness, &rng);
    int parent2 = tournament(slots, n, g->fitness, &rng);
    for (int tries = 0; parent2 == parent1 && tries < 8; ++tries)
        parent2 = tournament(slots, n, g->fitness, &rng);
    if (parent2 == parent1) {
        for (int k = 0; k < n; ++k)
            if (slots[k] != parent1) { parent2 = slots[k]; break; }
    }
    const int* genes1 = g->genes + (size_t)parent1 * L;
    const int* genes2 = g->genes + (size_t)parent2 * L;
    memcpy(child, genes1, sizeof(int) * L);
    if (orc_rng_next_coin(&rng, g->crossover_rate)) {
        int a = orc_rng_next_index(&rng, L + 1);
        int b = orc_rng_next_index(&rng, L + 1);
        while (b == a) b = orc_rng_next_index(&rng, L + 1);
        int lo = a < b ? a : b, hi = a < b ? b : a;
        for (int i = lo; i < hi; ++i) child[i] = genes2[i];
    }
    for (int i = 0; i < L; ++i)
        if (orc_rng_next_coin(&rng, g->mutation_rate))
            child[i] = orc_rng_next_index(&rng, inst->machines_per_stage[i % inst->num_stages]);
    if (draws) {  /* state = seed + n * gamma (mod 2^64); gamma is odd, so n = delta * gamma^-1 */
        uint64_t inv = GAMMA;
        for (int it = 0; it < 6; ++it) inv *= 2 - GAMMA * inv;
        *draws = (rng - stream_seed) * inv;
    }
    orc_report rep;
    orc_score(inst, child, g->emax, &rep, NULL, NULL, NULL, NULL, NULL);
    if (rep.fitness > g->fitness[index]) {
        *fit = rep.fitness;
        *obj = rep.objective;
        return 1;
    }
    *fit = g->fitness[index];
    *obj = g->objective[index];
    return 0;
}

void orc_cellular_step(orc_cellular* g) { /* :164-182 */
    const int L = g->inst->num_jobs * g->inst->num_stages;
    const int n = g->size;
    int* children = (int*)malloc(sizeof(int) * (size_t)n * L);
    double* fit = (double*)malloc(sizeof(double) * n);
    double* obj = (double*)malloc(sizeof(double) * n);
    char* replaced = (char*)malloc(n);
    const uint64_t gen_seed = orc_derive_seed(g->island_seed, g->generation + 1);
    for (int i = 0; i < n; ++i)
        replaced[i] = (char)orc_cellular_candidate(g, i, orc_derive_seed(gen_seed, (uint64_t)i),
                                                   children + (size_t)i * L, &fit[i], &obj[i]);
    for (int i = 0; i < n; ++i) {
        if (!replaced[i]) continue;
        memcpy(g->genes + (size_t)i * L, children + (size_t)i * L, sizeof(int) * L);
        g->fitness[i] = fit[i];
        g->objective[i] = obj[i];
    }
    ++g->generation;
    free(children); free(fit); free(obj); free(replaced);
}

int orc_cellular_best_index(const orc_cellular* g) { /* :184-189 */
    int best = 0;
    for (int i = 1; i < g->size; ++i)
        if (g->fitness[i] > g->fitness[best]) best = i;
    return best;
}

void orc_cellular_install(orc_cellular* g, int index, const int* genes, double fit, double obj) {
    /* :191-195 */
    const int L = g->inst->num_jobs * g->inst->num_stages;
    memcpy(g->genes + (size_t)index * L, genes, sizeof(int) * L);
    g->fitness[index] = fit;
    g->objective[index] = obj;
}

/* ---------------------------------------------------- Pseudo island (pseudo.cpp:11-113) */
int orc_pair_step(const uint8_t* a, const uint8_t* b, int nbits, uint64_t* rng,
                  double crossover_rate, uint8_t* child1, uint8_t* child2) { /* :11-29 */
    if (!orc_rng_next_coin(rng, crossover_rate)) {
        memcpy(child1, a, nbits);
        memcpy(child2, b, nbits);
        return 0;
    }
    uint64_t word = 0;
    for (int i = 0; i < nbits; ++i) {
        if (i % 64 == 0) word = orc_rng_next_u64(rng);
        int take_a = (int)((word >> (i % 64)) & 1u);
        child1[i] = take_a ? a[i] : b[i];
        child2[i] = take_a ? b[i] : a[i];
    }
    return 1;
}

static void consider_for_archive(orc_pseudo* p, const uint8_t* c, double fit, double obj) {
    /* :106-113 */
    if (fit > p->archive_fitness) {
        memcpy(p->archive, c, p->layout.total_bits);
        p->archive_fitness = fit;
        p->archive_objective = obj;
    }
}

static void score_bits(const orc_pseudo* p, const uint8_t* bits, int* scratch, orc_report* rep) {
    orc_bits_to_int(&p->layout, p->inst->machines_per_stage, bits, scratch);
    orc_score(p->inst, scratch, p->emax, rep, NULL, NULL, NULL, NULL, NULL);
}

orc_pseudo* orc_pseudo_new(const orc_instance* inst, double emax, int population,
                           double crossover_rate, uint64_t island_seed) { /* :31-57 */
    if (population < 2 || population % 2 != 0) return NULL;
    orc_pseudo* p = (orc_pseudo*)calloc(1, sizeof(orc_pseudo));
    p->inst = inst;
    p->emax = emax;
    orc_bit_layout_for(inst, &p->layout);
    p->size = population;
    p->crossover_rate = crossover_rate;
    p->island_seed = island_seed;
    const int nb = p->layout.total_bits;
    const int L = inst->num_jobs * inst->num_stages;
    p->members = (uint8_t*)malloc((size_t)population * nb);
    p->fitness = (double*)malloc(sizeof(double) * population);
    p->objective = (double*)malloc(sizeof(double) * population);
    p->archive = (uint8_t*)calloc(nb > 0 ? nb : 1, 1);
    p->archive_fitness = -1.0;
    p->archive_objective = 0.0;
    int* genes = (int*)malloc(sizeof(int) * L);
    uint64_t rng = island_seed;
    for (int q = 0; q < population / 2; ++q) {
        uint8_t* a = p->members + (size_t)(2 * q) * nb;
        uint8_t* b = p->members + (size_t)(2 * q + 1) * nb;
        orc_random_int_chromosome(inst, &rng, genes);
        orc_int_to_bits(&p->layout, inst->machines_per_stage, genes, a);
        for (int i = 0; i < nb; ++i) b[i] = a[i] ^ 1u;
    }
    for (int i = 0; i < population; ++i) {
        orc_report rep;
        score_bits(p, p->members + (size_t)i * nb, genes, &rep);
        p->fitness[i] = rep.fitness;
        p->objective[i] = rep.objective;
        consider_for_archive(p, p->members + (size_t)i * nb, p->fitness[i], p->objective[i]);
    }
    free(genes);
    return p;
}

void orc_pseudo_free(orc_pseudo* p) {
    if (!p) return;
    free(p->members); free(p->fitness); free(p->objective); free(p->archive); free(p);
}

void orc_pseudo_step(orc_pseudo* p) { /* :59-89 */
    const int pairs = p->size / 2;
    const int nb = p->layout.total_bits;
    const int L = p->inst->num_jobs * p->inst->num_stages;
    const uint64_t gen_seed = orc_derive_seed(p->island_seed, p->generation + 1);
    char* changed = (char*)calloc(pairs > 0 ? pairs : 1, 1);
    uint8_t* c1 = (uint8_t*)malloc(nb > 0 ? nb : 1);
    uint8_t* c2 = (uint8_t*)malloc(nb > 0 ? nb : 1);
    int* genes = (int*)malloc(sizeof(int) * L);
    for (int q = 0; q < pairs; ++q) {
        uint64_t rng = orc_derive_seed(gen_seed, (uint64_t)q);
        uint8_t* a = p->members + (size_t)(2 * q) * nb;
        uint8_t* b = p->members + (size_t)(2 * q + 1) * nb;
        if (!orc_pair_step(a, b, nb, &rng, p->crossover_rate, c1, c2)) continue;
        orc_report r1, r2;
        score_bits(p, c1, genes, &r1);
        score_bits(p, c2, genes, &r2);
        memcpy(a, c1, nb);
        memcpy(b, c2, nb);
        p->fitness[2 * q] = r1.fitness;
        p->objective[2 * q] = r1.objective;
        p->fitness[2 * q + 1] = r2.fitness;
        p->objective[2 * q + 1] = r2.objective;
        changed[q] = 1;
    }
    for (int q = 0; q < pairs; ++q) {
        if (!changed[q]) continue;
        consider_for_archive(p, p->members + (size_t)(2 * q) * nb, p->fitness[2 * q], p->objective[2 * q]);
        consider_for_archive(p, p->members + (size_t)(2 * q + 1) * nb, p->fitness[2 * q + 1],
                             p->objective[2 * q + 1]);
    }
    ++p->generation;
    free(changed); free(c1); free(c2); free(genes);
}

int orc_pseudo_best_index(const orc_pseudo* p) { /* :91-96 */
    int best = 0;
    for (int i = 1; i < p->size; ++i)
        if (p->fitness[i] > p->fitness[best]) best = i;
    return best;
}

void orc_pseudo_install(orc_pseudo* p, int index, const uint8_t* bits, double fit, double obj) {
    /* :98-104 */
    memcpy(p->members + (size_t)index * p->layout.total_bits, bits, p->layout.total_bits);
    p->fitness[index] = fit;
    p->objective[index] = obj;
    consider_for_archive(p, bits, fit, obj);
}

/* --------------------------------------------------------- Migration (migration.cpp) */
double orc_compute_beta(double fit_a, double fit_b) { /* :9-14 */
    if (fit_a == fit_b) return 1.0;
    return fit_a < fit_b ? fit_a / fit_b : fit_b / fit_a;
}

double orc_compute_alpha(double beta, double theta) { /* :16-19 */
    double rate = 1.0 - beta;
    return rate < theta ? rate : 0.0;
}

void orc_decide(double fit_a, double fit_b, double theta, int island_population, double* beta,
                double* alpha, int* direction, int* migrants) { /* :21-36 */
    *beta = orc_compute_beta(fit_a, fit_b);
    *alpha = orc_compute_alpha(*beta, theta);
    *migrants = (int)floor(*alpha * island_population);
    if (*migrants <= 0 || fit_a == fit_b) {
        *direction = 0;
        *migrants = 0;
        return;
    }
    *direction = fit_a > fit_b ? 1 : 2;
}

void orc_migrate_cellular_to_pseudo(const orc_cellular* from, orc_pseudo* to, int k) { /* :47-57 */
    const int L = from->inst->num_jobs * from->inst->num_stages;
    int* best = (int*)malloc(sizeof(int) * from->size);
    int* worst = (int*)malloc(sizeof(int) * to->size);
    uint8_t* bits = (uint8_t*)malloc(to->layout.total_bits > 0 ? to->layout.total_bits : 1);
    orc_sort_island(from->fitness, from->size, best);
    orc_sort_island(to->fitness, to->size, worst);
    for (int i = 0; i < k; ++i) {
        int src = best[i];
        int dst = worst[to->size - 1 - i];
        orc_int_to_bits(&to->layout, to->inst->machines_per_stage, from->genes + (size_t)src * L, bits);
        orc_pseudo_install(to, dst, bits, from->fitness[src], from->objective[src]);
    }
    free(best); free(worst); free(bits);
}

void orc_migrate_pseudo_to_cellular(const orc_pseudo* from, orc_cellular* to, int k) { /* :59-69 */
    const int L = to->inst->num_jobs * to->inst->num_stages;
    int* best = (int*)malloc(sizeof(int) * from->size);
    int* worst = (int*)malloc(sizeof(int) * to->size);
    int* genes = (int*)malloc(sizeof(int) * L);
    orc_sort_island(from->fitness, from->size, best);
    orc_sort_island(to->fitness, to->size, worst);
    for (int i = 0; i < k; ++i) {
        int src = best[i];
        int dst = worst[to->size - 1 - i];
        orc_bits_to_int(&from->layout, from->inst->machines_per_stage,
                        from->members + (size_t)src * from->layout.total_bits, genes);
        orc_cellular_install(to, dst, genes, from->fitness[src], from->objective[src]);
    }
    free(best); free(worst); free(genes);
}

/* --------------------------------------------------------- Solver (solver.cpp:39-198) */
static int validate_config(const orc_run_config* c) { /* solver.cpp:39-70 */
    if (c->generations < 1 || c->migration_gap < 1) return -1;
    if (c->theta < 0.0 || c->theta > 1.0) return -1;
    if (c->cellular_crossover < 0.0 || c->cellular_crossover > 1.0) return -1;
    if (c->cellular_mutation < 0.0 || c->cellular_mutation > 1.0) return -1;
    if (c->pseudo_crossover < 0.0 || c->pseudo_crossover > 1.0) return -1;
    if (c->mode == 0 && (c->population < 8 || c->population % 4 != 0)) return -1;
    if (c->mode == 1 && c->population < 4) return -1;
    if (c->mode == 2 && (c->population < 2 || c->population % 2 != 0)) return -1;
    return 0;
}

int orc_run(const orc_run_config* cfg, const orc_instance* inst, orc_run_result* out) {
    if (validate_config(cfg) != 0) return -1;
    memset(out, 0, sizeof(*out));
    const int L = inst->num_jobs * inst->num_stages;
    out->emax = orc_estimate_emax(inst);
    const int island_size = cfg->mode == 0 ? cfg->population / 2 : cfg->population;
    const uint64_t budget = (uint64_t)cfg->generations;
    const int want_c = cfg->mode != 2, want_p = cfg->mode != 1;
    orc_cellular* grid = NULL;
    orc_pseudo* pairs = NULL;
    if (want_c) {
        int w = cfg->grid_w, h = cfg->grid_h;
        if (w > 0 || h > 0) {
            if (w * h != island_size || w < 2 || h < 2) return -1;
        } else if (orc_grid_shape_for(island_size, &w, &h) != 0) {
            return -1;
        }
        grid = orc_cellular_new(inst, out->emax, w, h, cfg->radius, cfg->cellular_crossover,
                                cfg->cellular_mutation, orc_derive_seed(cfg->seed, 0), NULL);
    }
    if (want_p)
        pairs = orc_pseudo_new(inst, out->emax, island_size, cfg->pseudo_crossover,
                               orc_derive_seed(cfg->seed, 1));
    out->trace_combined = (double*)calloc(budget, sizeof(double));
    if (want_c) out->trace_a = (double*)calloc(budget, sizeof(double));
    if (want_p) out->trace_b = (double*)calloc(budget, sizeof(double));
    int cap = 16;
    out->mig_generation = (uint64_t*)malloc(sizeof(uint64_t) * cap);
    out->mig_beta = (double*)malloc(sizeof(double) * cap);
    out->mig_alpha = (double*)malloc(sizeof(double) * cap);
    out->mig_direction = (int*)malloc(sizeof(int) * cap);
    out->mig_migrants = (int*)malloc(sizeof(int) * cap);

    const int both = want_c && want_p;
    uint64_t done = 0;
    const uint64_t gap = (uint64_t)cfg->migration_gap;
    while (done < budget) {
        uint64_t stop = (done / gap + 1) * gap;
        if (stop > budget) stop = budget;
        if (want_c)
            for (uint64_t g = done + 1; g <= stop; ++g) {
                orc_cellular_step(grid);
                out->trace_a[g - 1] = grid->objective[orc_cellular_best_index(grid)];
            }
        if (want_p)
            for (uint64_t g = done + 1; g <= stop; ++g) {
                orc_pseudo_step(pairs);
                out->trace_b[g - 1] = pairs->archive_objective;
            }
        done = stop;
        if (both && done < budget && done % gap == 0) {
            double fit_a = grid->fitness[orc_cellular_best_index(grid)];
            double fit_b = cfg->pseudo_fit_from_archive ? pairs->archive_fitness
                                                        : pairs->fitness[orc_pseudo_best_index(pairs)];
            double beta, alpha;
            int direction, migrants;
            orc_decide(fit_a, fit_b, cfg->theta, island_size, &beta, &alpha, &direction, &migrants);
            if (direction != 0) {
                if (direction == 1) orc_migrate_cellular_to_pseudo(grid, pairs, migrants);
                else orc_migrate_pseudo_to_cellular(pairs, grid, migrants);
                if (out->num_migrations == cap) {
                    cap *= 2;
                    out->mig_generation = (uint64_t*)realloc(out->mig_generation, sizeof(uint64_t) * cap);
                    out->mig_beta = (double*)realloc(out->mig_beta, sizeof(double) * cap);
                    out->mig_alpha = (double*)realloc(out->mig_alpha, sizeof(double) * cap);
                    out->mig_direction = (int*)realloc(out->mig_direction, sizeof(int) * cap);
                    out->mig_migrants = (int*)realloc(out->mig_migrants, sizeof(int) * cap);
                }
                int e = out->num_migrations++;
                out->mig_generation[e] = done;
                out->mig_beta[e] = beta;
                out->mig_alpha[e] = alpha;
                out->mig_direction[e] = direction;
                out->mig_migrants[e] = migrants;
                out->trace_a[done - 1] = grid->objective[orc_cellular_best_index(grid)];
                out->trace_b[done - 1] = pairs->archive_objective;
            }
        }
    }
    for (uint64_t g = 0; g < budget; ++g) {
        if (!both) out->trace_combined[g] = want_c ? out->trace_a[g] : out->trace_b[g];
        else out->trace_combined[g] = std_min(out->trace_a[g], out->trace_b[g]);
    }
    double fit_a = want_c ? grid->fitness[orc_cellular_best_index(grid)] : -1.0;
    double fit_b = want_p ? pairs->archive_fitness : -1.0;
    out->best_chromosome = (int*)malloc(sizeof(int) * L);
    if (want_c && fit_a >= fit_b) {
        memcpy(out->best_chromosome, grid->genes + (size_t)orc_cellular_best_index(grid) * L, sizeof(int) * L);
    } else {
        orc_bits_to_int(&pairs->layout, inst->machines_per_stage, pairs->archive, out->best_chromosome);
    }
    orc_report rep;
    orc_score(inst, out->best_chromosome, out->emax, &rep, NULL, NULL, NULL, NULL, NULL);
    out->best_objective = rep.objective;
    out->best_fitness = rep.fitness;
    out->best_makespan = rep.makespan;
    out->best_tardiness = rep.total_tardiness;
    orc_cellular_free(grid);
    orc_pseudo_free(pairs);
    return 0;
}

void orc_run_result_free(orc_run_result* r) {
    free(r->best_chromosome); free(r->trace_combined); free(r->trace_a); free(r->trace_b);
    free(r->mig_generation); free(r->mig_beta); free(r->mig_alpha); free(r->mig_direction);
    free(r->mig_migrants);
    memset(r, 0, sizeof(*r));
}
