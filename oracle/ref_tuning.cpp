// ref_tuning.cpp — definitions for the reference's tuning declarations.
//
// TEST INFRASTRUCTURE ONLY (oracle/_ref).  The reference declares these in
// proj/include/f2la/tuning.hpp:11-41 but ships no definition, so any TU that
// instantiates f2la::m4rm_mult fails to link (m4rm.hpp:182).  The formulas
// follow SPEC.md:404-434 (module `tuning`).
#include "f2la/tuning.hpp"

#include <cmath>
#include <stdexcept>

namespace f2la::tuning {

void CostModel::validate() const {                       // tuning.hpp:17
    if (table_size < 2 || table_size > word_bits)
        throw std::invalid_argument("CostModel: need 2 <= c <= b");
    if (!(xor_cost > 0.0) || !(popcount_cost > 0.0))
        throw std::invalid_argument("CostModel: costs must be positive");
}

double m4rm_cost(unsigned b, unsigned c, double n) {     // tuning.hpp:22
    return (double(b) / double(c)) * (std::ldexp(1.0, int(c)) - 1.0 + n);
}

unsigned optimal_table_size(unsigned b, double n) {      // tuning.hpp:26
    const unsigned hi = b < 16 ? b : 16;
    unsigned best = 2;
    double best_cost = m4rm_cost(b, 2, n);
    for (unsigned c = 3; c <= hi; ++c) {
        const double v = m4rm_cost(b, c, n);
        if (v < best_cost) { best_cost = v; best = c; }
    }
    return best;
}

std::size_t strassen_threshold(unsigned c) {             // tuning.hpp:30
    return 44 * std::size_t(c) + 6 * ((std::size_t(1) << c) - 1);
}

double predicted_decomposition_cost(double n, unsigned b, unsigned c, RankRegime regime) {
    const double d = regime == RankRegime::full ? 3.0 : 2.0;  // tuning.hpp:32-37
    return n * n * n / (d * double(b) * double(c));
}

double word_size_cost_ratio(double xor_b, double xor_2b) {   // tuning.hpp:41
    return 2.0 * (xor_b / xor_2b);
}

}  // namespace f2la::tuning
