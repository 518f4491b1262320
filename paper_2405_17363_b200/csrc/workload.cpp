// workload.cpp -- synthetic CB05-shaped Newton systems (see
// include/blockcells_workload.h for the reference functions restated).
// Input synthesis only: not on the solver path.
#include "blockcells_workload.h"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <new>
#include <random>
#include <thread>
#include <vector>

namespace {

constexpr double kReferenceTemperature = 300.0;  // mechanism.cpp:19-26
constexpr double kSurfacePressure = 1000.0;
constexpr double kTopPressure = 100.0;
constexpr double kDryAdiabatKappa = 0.2854;
constexpr double kRateCoeffLo = 1e-6;
constexpr double kRateCoeffHi = 1e2;
constexpr double kTempExponentSpan = 2.0;
constexpr double kEmissionFraction = 0.1;

enum Kind { Emission, Unimolecular, Bimolecular };

struct Reaction {
    Kind kind;
    std::vector<int64_t> reactants, products;
    double rate_coeff, temp_exponent;
};

// mechanism.cpp:31-34: top 53 bits of the mt19937_64 draw.
double uniform01(std::mt19937_64& rng) { return static_cast<double>(rng() >> 11) * 0x1.0p-53; }

int64_t uniform_index(std::mt19937_64& rng, int64_t n) {
    return std::min(static_cast<int64_t>(uniform01(rng) * static_cast<double>(n)), n - 1);
}

// mechanism.cpp:40-58: `count` distinct species from the pool minus
// `exclude` (the whole range when the pool would be too small).
std::vector<int64_t> pick_species(std::mt19937_64& rng, int64_t n, int64_t count,
                                  const std::vector<int64_t>& exclude) {
    std::vector<int64_t> pool;
    for (int64_t s = 0; s < n; ++s)
        if (std::find(exclude.begin(), exclude.end(), s) == exclude.end()) pool.push_back(s);
    if (static_cast<int64_t>(pool.size()) < count) {
        pool.resize(n);
        for (int64_t s = 0; s < n; ++s) pool[s] = s;
    }
    std::vector<int64_t> picked;
    for (int64_t i = 0; i < count; ++i) {
        const int64_t at = uniform_index(rng, static_cast<int64_t>(pool.size()));
        picked.push_back(pool[at]);
        pool.erase(pool.begin() + at);
    }
    return picked;
}

struct Stamp {
    int64_t slot;
    double sign;
    int64_t diff_pos;
};

}  // namespace

struct bcw_mechanism {
    int64_t species = 0;
    std::vector<Reaction> reactions;
    std::vector<int32_t> row_ptr, col_idx;
    std::vector<std::vector<Stamp>> stamps;
    std::vector<int64_t> diag;
};

namespace {

void build_tables(bcw_mechanism& m) {
    const int64_t n = m.species;
    // mechanism.cpp:176-197: full diagonal + every reactant coupling, sorted
    // and de-duplicated (from_triplets, csr.cpp:21-61).
    std::vector<std::pair<int64_t, int64_t>> rc;
    for (int64_t i = 0; i < n; ++i) rc.push_back({i, i});
    for (const Reaction& r : m.reactions)
        for (int64_t col : r.reactants) {
            for (int64_t row : r.reactants) rc.push_back({row, col});
            for (int64_t row : r.products) rc.push_back({row, col});
        }
    std::sort(rc.begin(), rc.end());
    rc.erase(std::unique(rc.begin(), rc.end()), rc.end());
    m.row_ptr.assign(n + 1, 0);
    m.col_idx.clear();
    for (const auto& [row, col] : rc) {
        m.col_idx.push_back(static_cast<int32_t>(col));
        m.row_ptr[row + 1]++;
    }
    for (int64_t i = 0; i < n; ++i) m.row_ptr[i + 1] += m.row_ptr[i];

    auto slot_of = [&](int64_t row, int64_t col) {  // mechanism.cpp:199-206
        const auto b = m.col_idx.begin() + m.row_ptr[row];
        const auto e = m.col_idx.begin() + m.row_ptr[row + 1];
        return static_cast<int64_t>(std::lower_bound(b, e, static_cast<int32_t>(col)) -
                                    m.col_idx.begin());
    };
    m.stamps.assign(m.reactions.size(), {});
    for (std::size_t j = 0; j < m.reactions.size(); ++j) {  // mechanism.cpp:208-218
        const Reaction& r = m.reactions[j];
        for (std::size_t pos = 0; pos < r.reactants.size(); ++pos) {
            const int64_t col = r.reactants[pos];
            for (int64_t row : r.reactants)
                m.stamps[j].push_back({slot_of(row, col), -1.0, static_cast<int64_t>(pos)});
            for (int64_t row : r.products)
                m.stamps[j].push_back({slot_of(row, col), +1.0, static_cast<int64_t>(pos)});
        }
    }
    m.diag.assign(n, 0);  // simulate.cpp:15-26 diagonal_slots
    for (int64_t i = 0; i < n; ++i)
        for (int64_t j = m.row_ptr[i]; j < m.row_ptr[i + 1]; ++j)
            if (m.col_idx[j] == i) {
                m.diag[i] = j;
                break;
            }
}

// mechanism.cpp:152-170
void conditions(int64_t c, int64_t total, int mode, double* p, double* t, double* e) {
    if (mode == BCW_MODE_IDEAL) {
        *p = kSurfacePressure;
        *t = kReferenceTemperature;
        *e = 1.0;
        return;
    }
    const double fraction =
        total == 1 ? 0.0 : static_cast<double>(c) / static_cast<double>(total - 1);
    *p = kSurfacePressure - (kSurfacePressure - kTopPressure) * fraction;
    *e = 1.0 - fraction;
    *t = kReferenceTemperature * std::pow(*p / kSurfacePressure, kDryAdiabatKappa);
}

// mechanism.cpp:221-233
void rates_for(const bcw_mechanism& m, int64_t c, int64_t total, int mode, double* rates) {
    double p, t, e;
    conditions(c, total, mode, &p, &t, &e);
    for (std::size_t j = 0; j < m.reactions.size(); ++j) {
        const Reaction& r = m.reactions[j];
        double k = r.rate_coeff * std::pow(t / kReferenceTemperature, r.temp_exponent);
        if (r.kind == Emission) k *= e;
        rates[j] = k;
    }
}

template <class F>
void parallel_for(int64_t count, int threads, F&& f) {
    int hw = static_cast<int>(std::thread::hardware_concurrency());
    if (threads <= 0) threads = hw > 0 ? hw : 1;
    threads = static_cast<int>(std::min<int64_t>(threads, std::max<int64_t>(count, 1)));
    if (threads <= 1) {
        f(0, count);
        return;
    }
    std::vector<std::thread> pool;
    const int64_t chunk = (count + threads - 1) / threads;
    for (int w = 0; w < threads; ++w) {
        const int64_t b = w * chunk, e = std::min(count, b + chunk);
        if (b >= e) break;
        pool.emplace_back([&f, b, e] { f(b, e); });
    }
    for (auto& th : pool) th.join();
}

}  // namespace

extern "C" {

int bcw_mechanism_create(int64_t species, int64_t reactions, uint64_t seed, bcw_mechanism** out) {
    if (!out || species < 2 || reactions < 1) return -1;  // mechanism.cpp:119-120
    bcw_mechanism* m = new (std::nothrow) bcw_mechanism;
    if (!m) return -7;
    m->species = species;
    std::mt19937_64 rng(seed);
    for (int64_t i = 0; i < reactions; ++i) {  // mechanism.cpp:127-147
        Reaction r;
        const double kind_draw = uniform01(rng);
        r.kind = kind_draw < kEmissionFraction ? Emission
                 : kind_draw < 0.55            ? Unimolecular
                                               : Bimolecular;
        const int64_t n_reactants = r.kind == Emission ? 0 : r.kind == Unimolecular ? 1 : 2;
        r.reactants = pick_species(rng, species, n_reactants, {});
        const int64_t n_products = uniform01(rng) < 0.5 ? 1 : 2;
        r.products = pick_species(rng, species, n_products, r.reactants);
        const double log_lo = std::log10(kRateCoeffLo);
        const double log_hi = std::log10(kRateCoeffHi);
        r.rate_coeff = std::pow(10.0, log_lo + uniform01(rng) * (log_hi - log_lo));
        r.temp_exponent = (2.0 * uniform01(rng) - 1.0) * kTempExponentSpan;
        m->reactions.push_back(std::move(r));
    }
    build_tables(*m);
    *out = m;
    return 0;
}

// An arbitrary mechanism (a MechanismSpec given as flat arrays) with the same
// evaluator tables (mechanism.cpp:172-219).  kind: 0 emission, 1 unimolecular,
// 2 bimolecular.
int bcw_mechanism_from_reactions(int64_t species, int64_t reactions, const int32_t* kind,
                                 const int32_t* reactant_ptr, const int32_t* reactants,
                                 const int32_t* product_ptr, const int32_t* products, const double* rate_coeff,
                                 const double* temp_exponent, bcw_mechanism** out) {
    if (!out || species < 1 || reactions < 0 || (reactions > 0 && (!kind || !reactant_ptr || !product_ptr ||
                                                                   !rate_coeff || !temp_exponent)))
        return -1;
    bcw_mechanism* m = new (std::nothrow) bcw_mechanism;
    if (!m) return -7;
    m->species = species;
    for (int64_t j = 0; j < reactions; ++j) {
        Reaction r;
        r.kind = kind[j] == 0 ? Emission : kind[j] == 1 ? Unimolecular : Bimolecular;
        for (int32_t q = reactant_ptr[j]; q < reactant_ptr[j + 1]; ++q) r.reactants.push_back(reactants[q]);
        for (int32_t q = product_ptr[j]; q < product_ptr[j + 1]; ++q) r.products.push_back(products[q]);
        for (int64_t sp : r.reactants)
            if (sp < 0 || sp >= species) {
                delete m;
                return -1;
            }
        for (int64_t sp : r.products)
            if (sp < 0 || sp >= species) {
                delete m;
                return -1;
            }
        r.rate_coeff = rate_coeff[j];
        r.temp_exponent = temp_exponent[j];
        m->reactions.push_back(std::move(r));
    }
    build_tables(*m);
    *out = m;
    return 0;
}

void bcw_mechanism_destroy(bcw_mechanism* m) { delete m; }
int64_t bcw_species(const bcw_mechanism* m) { return m->species; }
int64_t bcw_reactions(const bcw_mechanism* m) { return static_cast<int64_t>(m->reactions.size()); }
int64_t bcw_nnz(const bcw_mechanism* m) { return static_cast<int64_t>(m->col_idx.size()); }

int bcw_pattern(const bcw_mechanism* m, int32_t* row_ptr, int32_t* col_idx) {
    if (row_ptr) std::memcpy(row_ptr, m->row_ptr.data(), sizeof(int32_t) * m->row_ptr.size());
    if (col_idx) std::memcpy(col_idx, m->col_idx.data(), sizeof(int32_t) * m->col_idx.size());
    return 0;
}

int bcw_newton_batch(const bcw_mechanism* m, int64_t first, int64_t count, int64_t total_cells,
                     int mode, double h, const double* y, const double* y_prev, double* values,
                     double* rhs, int threads) {
    if (!m || count < 0 || first < 0 || first + count > total_cells || !(h > 0.0)) return -1;
    const int64_t n = m->species, nnz = bcw_nnz(m);
    const int64_t nr = bcw_reactions(m);
    parallel_for(count, threads, [&](int64_t b, int64_t e) {
        std::vector<double> rates(nr), f(n), ones(n, 1.0);
        for (int64_t c = b; c < e; ++c) {
            const double* yc = y ? y + c * n : ones.data();
            const double* yp = y_prev ? y_prev + c * n : yc;
            rates_for(*m, first + c, total_cells, mode, rates.data());
            // rhs_into (mechanism.cpp:235-247)
            std::fill(f.begin(), f.end(), 0.0);
            for (int64_t j = 0; j < nr; ++j) {
                const Reaction& r = m->reactions[j];
                double rate = rates[j];
                for (int64_t s : r.reactants) rate *= yc[s];
                for (int64_t s : r.reactants) f[s] -= rate;
                for (int64_t s : r.products) f[s] += rate;
            }
            // jacobian_into (mechanism.cpp:249-267)
            double* v = values + c * nnz;
            std::fill(v, v + nnz, 0.0);
            for (int64_t j = 0; j < nr; ++j) {
                const Reaction& r = m->reactions[j];
                if (r.kind == Emission) continue;
                for (const Stamp& st : m->stamps[j]) {
                    double partial = rates[j];
                    for (std::size_t pos = 0; pos < r.reactants.size(); ++pos)
                        if (static_cast<int64_t>(pos) != st.diff_pos) partial *= yc[r.reactants[pos]];
                    v[st.slot] += st.sign * partial;
                }
            }
            // fill_newton_system (simulate.cpp:37-41)
            for (int64_t k = 0; k < nnz; ++k) v[k] = -h * v[k];
            for (int64_t i = 0; i < n; ++i) v[m->diag[i]] += 1.0;
            double* bb = rhs + c * n;
            for (int64_t i = 0; i < n; ++i) bb[i] = -(yc[i] - yp[i] - h * f[i]);
        }
    });
    return 0;
}

int bcw_rate_constants(const bcw_mechanism* m, int64_t first, int64_t count, int64_t total_cells,
                       int mode, double* rates, int threads) {
    if (!m || count < 0 || first < 0 || first + count > total_cells) return -1;
    const int64_t nr = bcw_reactions(m);
    parallel_for(count, threads, [&](int64_t b, int64_t e) {
        for (int64_t c = b; c < e; ++c) rates_for(*m, first + c, total_cells, mode, rates + c * nr);
    });
    return 0;
}

int64_t bcw_stamp_count(const bcw_mechanism* m) {
    int64_t s = 0;
    for (const auto& v : m->stamps) s += static_cast<int64_t>(v.size());
    return s;
}

int bcw_stamp_program(const bcw_mechanism* m, int32_t* stamp_ptr, int32_t* stamp_slot,
                      double* stamp_sign, int32_t* stamp_other, int32_t* reactant_ptr,
                      int32_t* reactants, int32_t* product_ptr, int32_t* products,
                      int32_t* diag_slot) {
    int32_t s = 0, rr = 0, pp = 0;
    stamp_ptr[0] = 0;
    reactant_ptr[0] = 0;
    product_ptr[0] = 0;
    for (std::size_t j = 0; j < m->reactions.size(); ++j) {
        const Reaction& r = m->reactions[j];
        if (r.kind != Emission) {
            for (const Stamp& st : m->stamps[j]) {
                stamp_slot[s] = static_cast<int32_t>(st.slot);
                stamp_sign[s] = st.sign;
                stamp_other[s] = r.reactants.size() == 2
                                     ? static_cast<int32_t>(r.reactants[1 - st.diff_pos])
                                     : -1;
                ++s;
            }
        }
        stamp_ptr[j + 1] = s;
        for (int64_t x : r.reactants) reactants[rr++] = static_cast<int32_t>(x);
        for (int64_t x : r.products) products[pp++] = static_cast<int32_t>(x);
        reactant_ptr[j + 1] = rr;
        product_ptr[j + 1] = pp;
    }
    for (int64_t i = 0; i < m->species; ++i) diag_slot[i] = static_cast<int32_t>(m->diag[i]);
    return 0;
}

}  // extern "C"
