// islands.cpp -- CellGrid / PairPopulation / migration over the device islands of the C ABI.
//
// Population state, breeding, evaluation, replacement, archive and migration transfers live on
// the GPU (kernels.cu K2-K6).  This file keeps the reference class API (proj/include/ffsga/
// cellular.hpp, pseudo.hpp, migration.hpp) and host mirrors of the spans it returns.
#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

#include "ffsga/cellular.hpp"
#include "ffsga/device.hpp"
#include "ffsga/errors.hpp"
#include "ffsga/migration.hpp"
#include "ffsga/pseudo.hpp"
#include "ffsga_cuda.h"

namespace ffsga {

namespace {
ffsga_cuda_cellular CH(void* h) { return static_cast<ffsga_cuda_cellular>(h); }
ffsga_cuda_pseudo PH(void* h) { return static_cast<ffsga_cuda_pseudo>(h); }
ffsga_cuda_instance IH(const std::shared_ptr<DeviceInstance>& d) { return static_cast<ffsga_cuda_instance>(d->handle()); }

std::vector<int> flatten(const std::vector<IntChromosome>& cells, int L) {
    std::vector<int> flat;
    flat.reserve((size_t)cells.size() * L);
    for (const auto& c : cells) {
        if ((int)c.genes.size() != L) throw ContractError("decode: assignment length must be num_jobs * num_stages");
        flat.insert(flat.end(), c.genes.begin(), c.genes.end());
    }
    return flat;
}
}  // namespace

// ------------------------------------------------------------------------------ torus helpers
std::vector<GridPos> neighborhood(GridPos pos, int width, int height, int radius) {
    // von Neumann ball of `radius` on the torus, centre excluded, rows dy = -r..r then
    // dx ascending (the slot order tournaments index into, cellular.cpp:12-27)
    if (pos.x < 0 || pos.x >= width || pos.y < 0 || pos.y >= height)
        throw ContractError("neighborhood: position off grid");
    if (radius < 1) throw ContractError("neighborhood: radius must be >= 1");
    auto wrap = [](int v, int n) { return ((v % n) + n) % n; };
    std::vector<GridPos> ring;
    for (int dy = -radius; dy <= radius; ++dy) {
        const int reach = radius - (dy < 0 ? -dy : dy);
        for (int dx = -reach; dx <= reach; ++dx)
            if (dx != 0 || dy != 0) ring.push_back({wrap(pos.x + dx, width), wrap(pos.y + dy, height)});
    }
    return ring;
}

std::vector<int> sort_island(std::span<const double> fitness) {
    std::vector<int> order(fitness.size());
    std::iota(order.begin(), order.end(), 0);
    std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return fitness[a] > fitness[b]; });
    return order;  // fitness descending, equal fitness by ascending index
}

std::pair<int, int> grid_shape_for(int population) {
    if (population < 4) throw ConfigError("cellular island needs a population of at least 4");
    int side = 1;
    for (int d = 1; (long long)d * d <= population; ++d)
        if (population % d == 0) side = d;
    if (side < 2)
        throw ConfigError("cellular population " + std::to_string(population) +
                          " has no grid factorization with both sides >= 2");
    return {population / side, side};
}

// ------------------------------------------------------------------------------ CellGrid
CellGrid::CellGrid(const Instance& inst, double emax, int population, CellularParams params, std::uint64_t seed,
                   std::optional<std::pair<int, int>> shape)
    : inst_(&inst), emax_(emax), params_(params), island_seed_(seed) {
    if (shape) {
        if (shape->first * shape->second != population)
            throw ConfigError("cellular grid shape does not match island population");
        if (shape->first < 2 || shape->second < 2) throw ConfigError("cellular grid sides must both be >= 2");
        width_ = shape->first;
        height_ = shape->second;
    } else {
        std::tie(width_, height_) = grid_shape_for(population);
    }
    create(nullptr);
}

CellGrid::CellGrid(const Instance& inst, double emax, std::vector<IntChromosome> cells, int width, int height,
                   CellularParams params, std::uint64_t seed)
    : inst_(&inst), emax_(emax), width_(width), height_(height), params_(params), island_seed_(seed) {
    if (width < 1 || height < 1 || (long long)width * height != (long long)cells.size())
        throw ConfigError("cellular grid shape does not match cell count");
    const std::vector<int> flat = flatten(cells, inst.num_genes());
    create(flat.data());
}

void CellGrid::create(const int* init_genes) {
    dev_ = DeviceInstance::get(*inst_, emax_);
    ffsga_cuda_cellular h = nullptr;
    check_status(ffsga_cuda_cellular_create(IH(dev_), width_, height_, params_.neighborhood_radius,
                                            params_.crossover_rate, params_.mutation_rate, island_seed_, init_genes, &h));
    handle_ = h;
    for (int i = 0; i < size(); ++i)
        for (const GridPos& p : neighborhood({i % width_, i / width_}, width_, height_, params_.neighborhood_radius))
            slots_.push_back(p.y * width_ + p.x);
    neighbors_per_cell_ = (int)(slots_.size() / size());
    cells_.resize(size());
    cell_fresh_.assign(size(), 0);
}

CellGrid::~CellGrid() {
    if (handle_) ffsga_cuda_cellular_destroy(CH(handle_));
}

void CellGrid::invalidate() const {
    fresh_ = false;
    std::fill(cell_fresh_.begin(), cell_fresh_.end(), 0);
}

void CellGrid::refresh() const {
    if (fresh_) return;
    fitness_.resize(size());
    objective_.resize(size());
    check_status(ffsga_cuda_cellular_read(CH(handle_), fitness_.data(), objective_.data()));
    fresh_ = true;
}

void CellGrid::step(int) {
    ffsga_cuda_cellular h = CH(handle_);
    check_status(ffsga_cuda_step(&h, 1, nullptr, 0, 1, nullptr, nullptr));
    invalidate();
}

CellGrid::Candidate CellGrid::cell_candidate(int index, Rng& rng) const {
    Candidate c;
    c.chromosome.genes.resize(inst_->num_genes());
    int replaced = 0;
    std::uint64_t used = 0;
    check_status(ffsga_cuda_cellular_candidate(CH(handle_), index, rng.state(), c.chromosome.genes.data(), &c.fitness,
                                               &c.objective, &replaced, &used));
    c.replaced = replaced != 0;
    for (std::uint64_t k = 0; k < used; ++k) rng.next_u64();  // leave the stream where compute_cell does
    return c;
}

std::uint64_t CellGrid::generation() const {
    std::uint64_t g = 0;
    check_status(ffsga_cuda_cellular_generation(CH(handle_), &g));
    return g;
}

std::span<const double> CellGrid::fitness() const {
    refresh();
    return fitness_;
}

std::span<const double> CellGrid::objective() const {
    refresh();
    return objective_;
}

const IntChromosome& CellGrid::cell(int index) const {
    if (index < 0 || index >= size()) throw ContractError("cell index out of range");
    if (!cell_fresh_[index]) {
        cells_[index].genes.resize(inst_->num_genes());
        check_status(ffsga_cuda_cellular_genes(CH(handle_), index, cells_[index].genes.data()));
        cell_fresh_[index] = 1;
    }
    return cells_[index];
}

int CellGrid::best_index() const {
    int i = 0;
    check_status(ffsga_cuda_cellular_best(CH(handle_), &i, nullptr, nullptr));
    return i;
}

double CellGrid::best_fitness() const {
    double f = 0;
    check_status(ffsga_cuda_cellular_best(CH(handle_), nullptr, &f, nullptr));
    return f;
}

double CellGrid::best_objective() const {
    double o = 0;
    check_status(ffsga_cuda_cellular_best(CH(handle_), nullptr, nullptr, &o));
    return o;
}

void CellGrid::install(int index, IntChromosome chromosome, double fitness, double objective) {
    if ((int)chromosome.genes.size() != inst_->num_genes())
        throw ContractError("install: chromosome length must be num_jobs * num_stages");
    check_status(ffsga_cuda_cellular_install(CH(handle_), index, chromosome.genes.data(), fitness, objective));
    invalidate();
}

// ------------------------------------------------------------------------------ pair step
PairStepResult pair_step(const BitChromosome& a, const BitChromosome& b, Rng& rng, double crossover_rate) {
    // host helper with the stream contract of pseudo.cpp:11-29 (coin, then one mask word per
    // 64 bits, bit i of the word picks parent a); PairPopulation::step runs the K4 kernel
    if (a.bits.size() != b.bits.size()) throw ContractError("pair_step: parents must share one layout");
    PairStepResult r;
    if (!rng.next_coin(crossover_rate)) {
        r.child1 = a;
        r.child2 = b;
        return r;
    }
    r.crossover_applied = true;
    const size_t n = a.bits.size();
    r.child1.bits.resize(n);
    r.child2.bits.resize(n);
    for (size_t base = 0; base < n; base += 64) {
        const std::uint64_t mask = rng.next_u64();
        const size_t top = std::min(n, base + 64);
        for (size_t i = base; i < top; ++i) {
            const bool from_a = (mask >> (i - base)) & 1u;
            r.child1.bits[i] = from_a ? a.bits[i] : b.bits[i];
            r.child2.bits[i] = from_a ? b.bits[i] : a.bits[i];
        }
    }
    return r;
}

// ------------------------------------------------------------------------------ PairPopulation
PairPopulation::PairPopulation(const Instance& inst, double emax, int population, PseudoParams params,
                               std::uint64_t seed)
    : inst_(&inst), emax_(emax), layout_(BitLayout::for_instance(inst)), params_(params), size_(population) {
    if (population < 2 || population % 2 != 0) throw ConfigError("pseudo island population must be even and >= 2");
    dev_ = DeviceInstance::get(inst, emax);
    ffsga_cuda_pseudo h = nullptr;
    check_status(ffsga_cuda_pseudo_create(IH(dev_), population, params.crossover_rate, seed, &h));
    handle_ = h;
}

PairPopulation::~PairPopulation() {
    if (handle_) ffsga_cuda_pseudo_destroy(PH(handle_));
}

void PairPopulation::invalidate() const { fresh_ = members_fresh_ = archive_fresh_ = false; }

void PairPopulation::refresh() const {
    if (fresh_) return;
    fitness_.resize(size_);
    objective_.resize(size_);
    check_status(ffsga_cuda_pseudo_read(PH(handle_), fitness_.data(), objective_.data()));
    fresh_ = true;
}

void PairPopulation::step(int) {
    ffsga_cuda_pseudo h = PH(handle_);
    check_status(ffsga_cuda_step(nullptr, 0, &h, 1, 1, nullptr, nullptr));
    invalidate();
}

std::uint64_t PairPopulation::generation() const {
    std::uint64_t g = 0;
    check_status(ffsga_cuda_pseudo_generation(PH(handle_), &g));
    return g;
}

std::span<const double> PairPopulation::fitness() const {
    refresh();
    return fitness_;
}

std::span<const double> PairPopulation::objective() const {
    refresh();
    return objective_;
}

const BitChromosome& PairPopulation::member(int index) const {
    if (index < 0 || index >= size_) throw ContractError("member index out of range");
    if (!members_fresh_) {
        std::vector<uint8_t> all((size_t)size_ * layout_.total_bits);
        check_status(ffsga_cuda_pseudo_member(PH(handle_), -1, all.data()));
        members_.resize(size_);
        for (int i = 0; i < size_; ++i)
            members_[i].bits.assign(all.begin() + (size_t)i * layout_.total_bits,
                                    all.begin() + (size_t)(i + 1) * layout_.total_bits);
        members_fresh_ = true;
    }
    return members_[index];
}

int PairPopulation::best_index() const {
    int i = 0;
    check_status(ffsga_cuda_pseudo_best(PH(handle_), &i, nullptr, nullptr));
    return i;
}

double PairPopulation::best_fitness() const {
    double f = 0;
    check_status(ffsga_cuda_pseudo_best(PH(handle_), nullptr, &f, nullptr));
    return f;
}

double PairPopulation::best_objective() const {
    double o = 0;
    check_status(ffsga_cuda_pseudo_best(PH(handle_), nullptr, nullptr, &o));
    return o;
}

const BitChromosome& PairPopulation::archive_chromosome() const {
    if (!archive_fresh_) {
        archive_.bits.assign(layout_.total_bits, 0);
        check_status(ffsga_cuda_pseudo_archive(PH(handle_), &archive_fitness_, &archive_objective_, archive_.bits.data()));
        if (archive_fitness_ < 0.0) archive_.bits.clear();  // nothing archived yet (pseudo.hpp:78)
        archive_fresh_ = true;
    }
    return archive_;
}

double PairPopulation::archive_fitness() const {
    archive_chromosome();
    return archive_fitness_;
}

double PairPopulation::archive_objective() const {
    archive_chromosome();
    return archive_objective_;
}

void PairPopulation::install(int index, BitChromosome chromosome, double fitness, double objective) {
    if ((int)chromosome.bits.size() != layout_.total_bits)
        throw ContractError("install: bit count does not match layout");
    check_status(ffsga_cuda_pseudo_install(PH(handle_), index, chromosome.bits.data(), fitness, objective));
    invalidate();
}

void step_islands(std::span<CellGrid* const> cells, std::span<PairPopulation* const> pseudos, int generations,
                  std::vector<std::vector<double>>* cell_traces, std::vector<std::vector<double>>* pseudo_traces) {
    std::vector<ffsga_cuda_cellular> ch;
    std::vector<ffsga_cuda_pseudo> ph;
    for (auto* c : cells) ch.push_back(CH(c->device_handle()));
    for (auto* p : pseudos) ph.push_back(PH(p->device_handle()));
    std::vector<double> tc(ch.size() * (size_t)std::max(generations, 0)), tp(ph.size() * (size_t)std::max(generations, 0));
    check_status(ffsga_cuda_step(ch.data(), (int)ch.size(), ph.data(), (int)ph.size(), generations,
                                 tc.empty() ? nullptr : tc.data(), tp.empty() ? nullptr : tp.data()));
    for (auto* c : cells) c->invalidate();
    for (auto* p : pseudos) p->invalidate();
    auto split = [generations](const std::vector<double>& flat, size_t n, std::vector<std::vector<double>>* out) {
        if (!out) return;
        out->assign(n, {});
        for (size_t i = 0; i < n; ++i)
            (*out)[i].assign(flat.begin() + i * generations, flat.begin() + (i + 1) * generations);
    };
    split(tc, ch.size(), cell_traces);
    split(tp, ph.size(), pseudo_traces);
}

// ------------------------------------------------------------------------------ migration
double compute_beta(double fit_a, double fit_b) {
    if (fit_a < 0.0 || fit_b < 0.0) throw ContractError("compute_beta: fitness values must be non-negative");
    if (fit_a == fit_b) return 1.0;
    return fit_a < fit_b ? fit_a / fit_b : fit_b / fit_a;  // smaller over larger
}

double compute_alpha(double beta, double theta) {
    const double rate = 1.0 - beta;
    return rate < theta ? rate : 0.0;
}

MigrationDecision decide(double fit_a, double fit_b, const MigrationPolicy& policy, int island_population) {
    if (island_population < 1) throw ContractError("decide: island population must be positive");
    MigrationDecision d;
    d.beta = compute_beta(fit_a, fit_b);
    d.alpha = compute_alpha(d.beta, policy.theta);
    const int k = static_cast<int>(std::floor(d.alpha * island_population));
    if (k <= 0 || fit_a == fit_b) return MigrationDecision{d.beta, d.alpha, MigrationDirection::none, 0};
    d.migrants = k;
    d.direction = fit_a > fit_b ? MigrationDirection::a_to_b : MigrationDirection::b_to_a;
    return d;
}

void migrate_cellular_to_pseudo(const CellGrid& from, PairPopulation& to, int k) {
    check_status(ffsga_cuda_migrate_cellular_to_pseudo(CH(from.device_handle()), PH(to.device_handle()), k));
    to.invalidate();
}

void migrate_pseudo_to_cellular(const PairPopulation& from, CellGrid& to, int k) {
    check_status(ffsga_cuda_migrate_pseudo_to_cellular(PH(from.device_handle()), CH(to.device_handle()), k));
    to.invalidate();
}

}  // namespace ffsga

namespace ffsga {
void* PairPopulation::device_handle() const { return handle_; }
}  // namespace ffsga
