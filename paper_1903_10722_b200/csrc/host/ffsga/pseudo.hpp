// pseudo.hpp -- complementary-pair island (API of proj/include/ffsga/pseudo.hpp:14-81).
// Members live on the GPU bit-packed (u64 words, LSB-first = the reference mask order);
// step() runs the K4 breed kernel, the K1 decoder and the K6 commit/archive kernel.
#pragma once

#include <cstdint>
#include <memory>
#include <span>
#include <vector>

#include "ffsga/chromosome.hpp"
#include "ffsga/instance.hpp"
#include "ffsga/model.hpp"
#include "ffsga/rng.hpp"

namespace ffsga {

struct PseudoParams {
    double crossover_rate = 0.75;
};

struct PairStepResult {
    BitChromosome child1;
    BitChromosome child2;
    bool crossover_applied = false;
};
// Mask crossover of one pair on an explicit stream (host helper for tests and callers).
PairStepResult pair_step(const BitChromosome& a, const BitChromosome& b, Rng& rng, double crossover_rate);

class PairPopulation {
  public:
    PairPopulation(const Instance& inst, double emax, int population, PseudoParams params, std::uint64_t island_seed);
    ~PairPopulation();
    PairPopulation(const PairPopulation&) = delete;
    PairPopulation& operator=(const PairPopulation&) = delete;

    void step(int workers = 1);

    int size() const { return size_; }
    int num_pairs() const { return size_ / 2; }
    std::uint64_t generation() const;
    const Instance& instance() const { return *inst_; }
    const BitLayout& layout() const { return layout_; }
    double emax() const { return emax_; }
    const PseudoParams& params() const { return params_; }

    std::span<const double> fitness() const;
    std::span<const double> objective() const;
    const BitChromosome& member(int index) const;

    int best_index() const;
    double best_fitness() const;
    double best_objective() const;

    const BitChromosome& archive_chromosome() const;
    double archive_fitness() const;
    double archive_objective() const;

    void install(int index, BitChromosome chromosome, double fitness, double objective);

    void* device_handle() const;
    void invalidate() const;

  private:
    void refresh() const;

    const Instance* inst_;
    double emax_;
    BitLayout layout_;
    PseudoParams params_;
    int size_ = 0;
    std::shared_ptr<DeviceInstance> dev_;
    void* handle_ = nullptr;
    mutable bool fresh_ = false, members_fresh_ = false, archive_fresh_ = false;
    mutable std::vector<double> fitness_, objective_;
    mutable std::vector<BitChromosome> members_;
    mutable BitChromosome archive_;
    mutable double archive_fitness_ = -1.0, archive_objective_ = 0.0;
};

class CellGrid;

// Advance every listed island `generations` times with one fused launch sequence per
// generation (the device form of the concurrent island segment, solver.cpp:126-139).
// Traces (optional) receive best_objective() / archive_objective() after each generation,
// [island][generation].  All islands must be built on the same instance and emax.
void step_islands(std::span<CellGrid* const> cells, std::span<PairPopulation* const> pseudos, int generations,
                  std::vector<std::vector<double>>* cell_traces = nullptr,
                  std::vector<std::vector<double>>* pseudo_traces = nullptr);

}  // namespace ffsga
