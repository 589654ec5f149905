// migration.hpp -- penetration-inspired migration (API of proj/include/ffsga/migration.hpp).
// decide() is the scalar policy (host); the transfers run on the GPU (K5).
#pragma once

#include "ffsga/cellular.hpp"
#include "ffsga/pseudo.hpp"

namespace ffsga {

struct MigrationPolicy {
    double theta = 1.0;
    int gap = 500;
};

enum class MigrationDirection { none, a_to_b, b_to_a };

struct MigrationDecision {
    double beta = 1.0;
    double alpha = 0.0;
    MigrationDirection direction = MigrationDirection::none;
    int migrants = 0;
};

double compute_beta(double fit_a, double fit_b);
double compute_alpha(double beta, double theta);
MigrationDecision decide(double fit_a, double fit_b, const MigrationPolicy& policy, int island_population);
void migrate_cellular_to_pseudo(const CellGrid& from, PairPopulation& to, int k);
void migrate_pseudo_to_cellular(const PairPopulation& from, CellGrid& to, int k);

}  // namespace ffsga
