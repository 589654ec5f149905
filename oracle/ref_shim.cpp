// ref_shim.cpp -- C-ABI shim over the UNMODIFIED reference library (TEST INFRASTRUCTURE).
//
// Compiled together with the reference sources in /root/reference/proj/src by
// oracle/Makefile, with -Dffsga=ffsga_ref so every reference symbol lives in ffsga_ref::,
// into oracle/_ref/libffsga_ref.so.  Used to pin the C restatement (ffsga_oracle.c) and as
// the "reference" CPU arm of bench.py.  Never linked into the product.
#include <cstdint>
#include <cstring>
#include <exception>
#include <memory>
#include <string>
#include <vector>

#include "ffsga/cellular.hpp"
#include "ffsga/chromosome.hpp"
#include "ffsga/generator.hpp"
#include "ffsga/io.hpp"
#include "ffsga/migration.hpp"
#include "ffsga/model.hpp"
#include "ffsga/parallel.hpp"
#include "ffsga/pseudo.hpp"
#include "ffsga/rng.hpp"
#include "ffsga/solver.hpp"
#include "oracle.hpp"

using namespace ffsga_ref;

namespace {
thread_local std::string g_err;
template <typename F>
int guard(F&& f) {
    try {
        f();
        return 0;
    } catch (const ContractError& e) {
        g_err = e.what();
        return 1;
    } catch (const ConfigError& e) {
        g_err = e.what();
        return 2;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 9;
    }
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_generate(int jobs, int stages, const int* machines, double weight, uint64_t seed,
                   int integer_times) {
    Instance* out = nullptr;
    guard([&] {
        GenParams p;
        p.num_jobs = jobs;
        p.num_stages = stages;
        p.machines_per_stage.assign(machines, machines + stages);
        p.weight = weight;
        p.seed = seed;
        p.integer_times = integer_times != 0;
        out = new Instance(generate(p));
    });
    return out;
}

void* ref_instance_new(int jobs, int stages, const int* machines, const double* proc,
                       const double* release, const double* due, double weight) {
    Instance* inst = new Instance();
    inst->num_jobs = jobs;
    inst->num_stages = stages;
    inst->machines_per_stage.assign(machines, machines + stages);
    inst->weight = weight;
    inst->finalize();
    inst->proc.assign(proc, proc + static_cast<size_t>(jobs) * inst->machines_total);
    inst->release.assign(release, release + jobs);
    inst->due.assign(due, due + jobs);
    return inst;
}

int ref_instance_validate(void* h) {
    return guard([&] { static_cast<Instance*>(h)->validate(); });
}

int ref_instance_machines_total(void* h) { return static_cast<Instance*>(h)->machines_total; }

void ref_instance_export(void* h, double* proc, double* release, double* due) {
    auto* inst = static_cast<Instance*>(h);
    std::memcpy(proc, inst->proc.data(), sizeof(double) * inst->proc.size());
    std::memcpy(release, inst->release.data(), sizeof(double) * inst->release.size());
    std::memcpy(due, inst->due.data(), sizeof(double) * inst->due.size());
}

void ref_instance_free(void* h) { delete static_cast<Instance*>(h); }

double ref_estimate_emax(void* h) { return estimate_emax(*static_cast<Instance*>(h)); }
double ref_mean_total_load(void* h) { return mean_total_load(*static_cast<Instance*>(h)); }

// Evaluator::score over a batch of job-major int32 chromosomes, parallel_chunks fan-out
// exactly as the islands use it (cellular.cpp:168-174).
int ref_score_batch(void* h, double emax, const int32_t* genes, int64_t n, double* obj,
                    double* fit, double* makespan, double* tard, int workers) {
    auto* inst = static_cast<Instance*>(h);
    const int L = inst->num_genes();
    return guard([&] {
        parallel_chunks(static_cast<int>(n), workers, [&](int lo, int hi) {
            Evaluator eval(*inst, emax);
            for (int i = lo; i < hi; ++i) {
                std::span<const int> g(genes + static_cast<size_t>(i) * L, L);
                ObjectiveReport r = eval.score(g);
                if (obj) obj[i] = r.objective;
                if (fit) fit[i] = r.fitness;
                if (makespan) makespan[i] = r.makespan;
                if (tard) tard[i] = r.total_tardiness;
            }
        });
    });
}

int ref_decode(void* h, const int32_t* genes, int* machine, double* start, double* completion) {
    auto* inst = static_cast<Instance*>(h);
    return guard([&] {
        std::vector<int> g(genes, genes + inst->num_genes());
        Schedule s = decode(*inst, g);
        std::memcpy(machine, s.machine.data(), sizeof(int) * s.machine.size());
        std::memcpy(start, s.start.data(), sizeof(double) * s.start.size());
        std::memcpy(completion, s.completion.data(), sizeof(double) * s.completion.size());
    });
}

double ref_oracle_simulate(void* h, const int32_t* genes) {
    auto* inst = static_cast<Instance*>(h);
    std::vector<int> g(genes, genes + inst->num_genes());
    return oracle::simulate(*inst, g).objective;
}

void ref_random_chromosomes(void* h, uint64_t base_seed, int64_t first, int64_t n, int32_t* out) {
    // chromosome i = random_int_chromosome(inst, Rng(derive_seed(base, first + i)))
    auto* inst = static_cast<Instance*>(h);
    const int L = inst->num_genes();
    for (int64_t i = 0; i < n; ++i) {
        Rng rng(derive_seed(base_seed, static_cast<uint64_t>(first + i)));
        IntChromosome c = random_int_chromosome(*inst, rng);
        std::memcpy(out + i * L, c.genes.data(), sizeof(int) * L);
    }
}

uint64_t ref_derive_seed(uint64_t base, uint64_t key) { return derive_seed(base, key); }

// ---- cellular island ------------------------------------------------------------------
void* ref_cellular_new(void* h, double emax, int population, int width, int height, int radius,
                       double xr, double mr, uint64_t seed) {
    CellGrid* g = nullptr;
    int st = guard([&] {
        CellularParams p{xr, mr, radius};
        std::optional<std::pair<int, int>> shape;
        if (width > 0) shape = std::make_pair(width, height);
        g = new CellGrid(*static_cast<Instance*>(h), emax, population, p, seed, shape);
    });
    return st == 0 ? g : nullptr;
}

void* ref_cellular_new_explicit(void* h, double emax, const int32_t* genes, int width, int height,
                                int radius, double xr, double mr, uint64_t seed) {
    auto* inst = static_cast<Instance*>(h);
    CellGrid* g = nullptr;
    int st = guard([&] {
        const int L = inst->num_genes();
        std::vector<IntChromosome> cells(static_cast<size_t>(width) * height);
        for (size_t i = 0; i < cells.size(); ++i)
            cells[i].genes.assign(genes + i * L, genes + (i + 1) * L);
        g = new CellGrid(*inst, emax, std::move(cells), width, height, CellularParams{xr, mr, radius},
                         seed);
    });
    return st == 0 ? g : nullptr;
}

void ref_cellular_free(void* g) { delete static_cast<CellGrid*>(g); }
void ref_cellular_step(void* g, int workers) { static_cast<CellGrid*>(g)->step(workers); }
int ref_cellular_size(void* g) { return static_cast<CellGrid*>(g)->size(); }
int ref_cellular_width(void* g) { return static_cast<CellGrid*>(g)->width(); }
int ref_cellular_height(void* g) { return static_cast<CellGrid*>(g)->height(); }
uint64_t ref_cellular_generation(void* g) { return static_cast<CellGrid*>(g)->generation(); }
int ref_cellular_best_index(void* g) { return static_cast<CellGrid*>(g)->best_index(); }

void ref_cellular_read(void* g, double* fit, double* obj, int32_t* genes) {
    auto* grid = static_cast<CellGrid*>(g);
    const int n = grid->size();
    for (int i = 0; i < n; ++i) {
        if (fit) fit[i] = grid->fitness()[i];
        if (obj) obj[i] = grid->objective()[i];
        if (genes) {
            const auto& c = grid->cell(i).genes;
            std::memcpy(genes + static_cast<size_t>(i) * c.size(), c.data(), sizeof(int) * c.size());
        }
    }
}

void ref_cellular_slots(void* g, int index, int* slots, int* count) {
    auto s = static_cast<CellGrid*>(g)->neighbor_slots(index);
    *count = static_cast<int>(s.size());
    for (size_t i = 0; i < s.size(); ++i) slots[i] = s[i];
}

int ref_cellular_candidate(void* g, int index, uint64_t stream_seed, int32_t* child, double* fit,
                           double* obj) {
    auto* grid = static_cast<CellGrid*>(g);
    Rng rng(stream_seed);
    CellGrid::Candidate c = grid->cell_candidate(index, rng);
    std::memcpy(child, c.chromosome.genes.data(), sizeof(int) * c.chromosome.genes.size());
    *fit = c.fitness;
    *obj = c.objective;
    return c.replaced ? 1 : 0;
}

void ref_cellular_install(void* g, int index, const int32_t* genes, double fit, double obj) {
    auto* grid = static_cast<CellGrid*>(g);
    IntChromosome c;
    c.genes.assign(genes, genes + grid->instance().num_genes());
    grid->install(index, std::move(c), fit, obj);
}

// ---- pseudo island ---------------------------------------------------------------------
void* ref_pseudo_new(void* h, double emax, int population, double xr, uint64_t seed) {
    PairPopulation* p = nullptr;
    int st = guard([&] {
        p = new PairPopulation(*static_cast<Instance*>(h), emax, population, PseudoParams{xr}, seed);
    });
    return st == 0 ? p : nullptr;
}
void ref_pseudo_free(void* p) { delete static_cast<PairPopulation*>(p); }
void ref_pseudo_step(void* p, int workers) { static_cast<PairPopulation*>(p)->step(workers); }
int ref_pseudo_size(void* p) { return static_cast<PairPopulation*>(p)->size(); }
int ref_pseudo_total_bits(void* p) { return static_cast<PairPopulation*>(p)->layout().total_bits; }
int ref_pseudo_best_index(void* p) { return static_cast<PairPopulation*>(p)->best_index(); }
uint64_t ref_pseudo_generation(void* p) { return static_cast<PairPopulation*>(p)->generation(); }

void ref_pseudo_read(void* p, double* fit, double* obj, uint8_t* bits) {
    auto* pop = static_cast<PairPopulation*>(p);
    const int nb = pop->layout().total_bits;
    for (int i = 0; i < pop->size(); ++i) {
        if (fit) fit[i] = pop->fitness()[i];
        if (obj) obj[i] = pop->objective()[i];
        if (bits) std::memcpy(bits + static_cast<size_t>(i) * nb, pop->member(i).bits.data(), nb);
    }
}

void ref_pseudo_archive(void* p, double* fit, double* obj, uint8_t* bits) {
    auto* pop = static_cast<PairPopulation*>(p);
    *fit = pop->archive_fitness();
    *obj = pop->archive_objective();
    if (bits && !pop->archive_chromosome().bits.empty())
        std::memcpy(bits, pop->archive_chromosome().bits.data(), pop->archive_chromosome().bits.size());
}

void ref_pseudo_install(void* p, int index, const uint8_t* bits, double fit, double obj) {
    auto* pop = static_cast<PairPopulation*>(p);
    BitChromosome b;
    b.bits.assign(bits, bits + pop->layout().total_bits);
    pop->install(index, std::move(b), fit, obj);
}

int ref_pair_step(const uint8_t* a, const uint8_t* b, int nbits, uint64_t seed, double xr,
                  uint8_t* c1, uint8_t* c2) {
    BitChromosome x, y;
    x.bits.assign(a, a + nbits);
    y.bits.assign(b, b + nbits);
    Rng rng(seed);
    PairStepResult r = pair_step(x, y, rng, xr);
    std::memcpy(c1, r.child1.bits.data(), nbits);
    std::memcpy(c2, r.child2.bits.data(), nbits);
    return r.crossover_applied ? 1 : 0;
}

// ---- migration ---------------------------------------------------------------------------
void ref_decide(double fa, double fb, double theta, int n, double* beta, double* alpha, int* dir,
                int* migrants) {
    MigrationDecision d = decide(fa, fb, MigrationPolicy{theta, 1}, n);
    *beta = d.beta;
    *alpha = d.alpha;
    *dir = static_cast<int>(d.direction);
    *migrants = d.migrants;
}
void ref_migrate_c2p(void* g, void* p, int k) {
    migrate_cellular_to_pseudo(*static_cast<CellGrid*>(g), *static_cast<PairPopulation*>(p), k);
}
void ref_migrate_p2c(void* p, void* g, int k) {
    migrate_pseudo_to_cellular(*static_cast<PairPopulation*>(p), *static_cast<CellGrid*>(g), k);
}

// ---- whole run --------------------------------------------------------------------------
struct RefRun {
    RunResult r;
    RunConfig c;
};

void* ref_run(void* h, int population, int generations, int gap, double theta, int mode,
              uint64_t seed, int workers, int serialized, double cx, double cm, double px,
              int pseudo_fit_from_archive) {
    RefRun* out = nullptr;
    guard([&] {
        RunConfig c;
        c.population = population;
        c.generations = generations;
        c.migration_gap = gap;
        c.theta = theta;
        c.mode = static_cast<RunMode>(mode);
        c.seed = seed;
        c.workers = workers;
        c.cellular.crossover_rate = cx;
        c.cellular.mutation_rate = cm;
        c.pseudo.crossover_rate = px;
        c.pseudo_fit_from_archive = pseudo_fit_from_archive != 0;
        auto* rr = new RefRun();
        rr->c = c;
        rr->r = serialized ? run_serialized(c, *static_cast<Instance*>(h)) : run(c, *static_cast<Instance*>(h));
        out = rr;
    });
    return out;
}

void ref_run_scalars(void* r, double* out5) {
    const RunResult& x = static_cast<RefRun*>(r)->r;
    out5[0] = x.best_objective;
    out5[1] = x.best_fitness;
    out5[2] = x.best_makespan;
    out5[3] = x.best_tardiness;
    out5[4] = x.emax;
}
int ref_run_num_migrations(void* r) { return static_cast<int>(static_cast<RefRun*>(r)->r.migrations.size()); }
void ref_run_migration(void* r, int i, uint64_t* gen, double* beta, double* alpha, int* dir, int* k) {
    const MigrationEvent& e = static_cast<RefRun*>(r)->r.migrations[i];
    *gen = e.generation;
    *beta = e.beta;
    *alpha = e.alpha;
    *dir = static_cast<int>(e.direction);
    *k = e.migrants;
}
void ref_run_traces(void* r, double* combined, double* a, double* b, int32_t* chromosome) {
    const RunResult& x = static_cast<RefRun*>(r)->r;
    std::memcpy(combined, x.trace_combined.data(), sizeof(double) * x.trace_combined.size());
    if (a && !x.trace_island_a.empty()) std::memcpy(a, x.trace_island_a.data(), sizeof(double) * x.trace_island_a.size());
    if (b && !x.trace_island_b.empty()) std::memcpy(b, x.trace_island_b.data(), sizeof(double) * x.trace_island_b.size());
    std::memcpy(chromosome, x.best_chromosome.genes.data(), sizeof(int) * x.best_chromosome.genes.size());
}
void ref_run_free(void* r) { delete static_cast<RefRun*>(r); }

// ---- file formats (io.cpp): result JSON, trace CSV, instance JSON ------------------------
int ref_save_result_json(void* r, const char* path) {
    return guard([&] { save_result_json(static_cast<RefRun*>(r)->r, static_cast<RefRun*>(r)->c, path); });
}
int ref_save_trace_csv(void* r, const char* path) {
    return guard([&] { save_trace_csv(static_cast<RefRun*>(r)->r, path); });
}
int ref_save_instance(void* h, const char* path) {
    return guard([&] { save_instance(*static_cast<Instance*>(h), path); });
}

}  // extern "C"
