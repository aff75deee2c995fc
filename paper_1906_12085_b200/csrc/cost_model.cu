// cost_model.cpp — the paper's modeled cost of one factorization (host only).
//
// Restates the published closed forms the reference evaluates in
// cost_model.cpp:30-113 (paper tables of flop and storage counts), used for
// the bench grid's model_flops / model_space_bytes columns (bench.cpp:109-121):
//
//   truncated             F = 2mn^2 + n^3 + n + mn
//                         S = 3n^2 + 3n + 2mn
//   randomized (l, i)     F = nl + (2i+2) mnl + l^2 (3m + n - 2l/3)
//                         S = mn + 3ml + 3nl + 2l^2
//   randomized, practical F = n^2/2 + 11/4 mn^2 + n^3/6          (l = n/2, i = 1)
//                         S = 9/2 mn + 3n^2
//   krylov (l, i)         w = (i+1) l
//                         F = nl + (3i+2) mnl + w^2 (m^2 + n^2 + 2m - 2w/3)
//                         S = mn + (3i+4) ml + (2i+3) nl + 2w^2
//   krylov, practical     F = n^2/2 + 5/2 mn^2 + 4 (m^2n^2 + 2mn^2 + n^4 - 2n^3/3)
//                         S = 9/2 mn + 9/2 n^2
//   krylov, per step      F = nl + (3i+2) mnl + w^2 (3m + n - 2w/3),  S as krylov
//
// Space counts 8-byte entries (input included); bytes are exactly 8 x entries.
// The printed "practical" forms are kept verbatim even where they do not
// follow from the general ones (the reference documents the same caveats,
// cost_model.hpp:22-43). Sums are evaluated left to right as written.
#include <cstdint>
#include <string>

#include "svdk_internal.h"

namespace svdk {

struct CostOut {
    double flops = 0.0, entries = 0.0;
};

namespace {

void need(bool ok, const char* model, uint64_t m, uint64_t n, uint64_t l, uint64_t i,
          uint64_t min_i) {
    if (!ok)
        fail(SVDK_E_PARAM, std::string(model) + ": outside the model's domain (m >= n >= l >= 1, i >= " +
                               std::to_string(min_i) + "): m=" + std::to_string(m) +
                               " n=" + std::to_string(n) + " l=" + std::to_string(l) +
                               " i=" + std::to_string(i));
}

}  // namespace

CostOut cost_model(int model, uint64_t m, uint64_t n, uint64_t l, uint64_t i) {
    const double M = static_cast<double>(m), N = static_cast<double>(n);
    const double L = static_cast<double>(l), It = static_cast<double>(i);
    const bool mn_ok = m >= n && n >= 1;
    const bool mnl_ok = m >= n && n >= l && l >= 1;
    CostOut c;
    switch (model) {
        case SVDK_COST_TRUNCATED:
            need(mn_ok, "truncated_cost", m, n, n, 0, 0);
            c.flops = 2.0 * M * N * N + N * N * N + N + M * N;
            c.entries = 3.0 * N * N + 3.0 * N + 2.0 * M * N;
            break;
        case SVDK_COST_RANDOMIZED:
            need(mnl_ok, "randomized_cost", m, n, l, i, 0);
            c.flops = N * L + (2.0 * It + 2.0) * M * N * L +
                      L * L * (3.0 * M + N - (2.0 / 3.0) * L);
            c.entries = M * N + 3.0 * M * L + 3.0 * N * L + 2.0 * L * L;
            break;
        case SVDK_COST_RANDOMIZED_PRACTICAL:
            need(mn_ok, "randomized_cost_practical", m, n, n, 1, 0);
            c.flops = N * N / 2.0 + 2.75 * M * N * N + N * N * N / 6.0;
            c.entries = 4.5 * M * N + 3.0 * N * N;
            break;
        case SVDK_COST_KRYLOV:
        case SVDK_COST_KRYLOV_PER_STEP: {
            need(mnl_ok && i >= 1, model == SVDK_COST_KRYLOV ? "krylov_cost" : "krylov_cost_per_step",
                 m, n, l, i, 1);
            const double w = (It + 1.0) * L;
            const double head = N * L + (3.0 * It + 2.0) * M * N * L;
            if (model == SVDK_COST_KRYLOV) {
                // the published total carries (i+1)^2 l^2 as one factor
                const double w2 = (It + 1.0) * (It + 1.0) * L * L;
                c.flops = head + w2 * (M * M + N * N + 2.0 * M - (2.0 / 3.0) * (It + 1.0) * L);
            } else {
                c.flops = head + w * w * (3.0 * M + N - (2.0 / 3.0) * w);
            }
            c.entries = M * N + (3.0 * It + 4.0) * M * L + (2.0 * It + 3.0) * N * L + 2.0 * w * w;
            break;
        }
        case SVDK_COST_KRYLOV_PRACTICAL:
            need(mn_ok, "krylov_cost_practical", m, n, n, 1, 0);
            c.flops = N * N / 2.0 + 2.5 * M * N * N +
                      4.0 * (M * M * N * N + 2.0 * M * N * N + N * N * N * N -
                             (2.0 / 3.0) * N * N * N);
            c.entries = 4.5 * M * N + 4.5 * N * N;
            break;
        default:
            fail(SVDK_E_PARAM, "cost_model: unknown model " + std::to_string(model));
    }
    return c;
}

}  // namespace svdk
