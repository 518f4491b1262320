// The shim's device-resident blockcells::b200::run_simulation (bc_simulate)
// against the reference's own blockcells::run_simulation (simulate.cpp, here
// driving the shim's GPU run_strategy): final states and every StepStats
// field but wall time, bit for bit; same errors.  TEST INFRASTRUCTURE (run on
// the GPU box by tests/test_simulate.py).
#include <cmath>
#include <cstring>
#include <optional>
#include <stdexcept>
#include <tuple>
#include <vector>

#include "blockcells/mechanism.hpp"
#include "blockcells/simulate.hpp"
#include "blockcells_b200_shim.hpp"
#include "doctest.h"

using namespace blockcells;

namespace {

bool same_bits(double a, double b) { return std::memcmp(&a, &b, sizeof a) == 0; }

void check_same(const SimulationResult& host, const SimulationResult& dev) {
    REQUIRE(host.per_step.size() == dev.per_step.size());
    REQUIRE(host.final_states.size() == dev.final_states.size());
    for (std::size_t i = 0; i < host.per_step.size(); ++i) {
        const StepStats &h = host.per_step[i], &d = dev.per_step[i];
        CHECK(h.step == d.step);
        CHECK(h.newton_iterations == d.newton_iterations);
        CHECK(h.iterations_effective == d.iterations_effective);
        CHECK(h.iterations_sum == d.iterations_sum);
        CHECK(same_bits(h.max_residual_rms, d.max_residual_rms));
        CHECK(h.breakdown_fallbacks == d.breakdown_fallbacks);
        CHECK(h.clip_events == d.clip_events);
    }
    std::size_t diff = 0;
    for (std::size_t c = 0; c < host.final_states.size(); ++c)
        for (std::size_t s = 0; s < host.final_states[c].concentrations.size(); ++s)
            diff += !same_bits(host.final_states[c].concentrations[s], dev.final_states[c].concentrations[s]);
    CHECK(diff == 0);
}

SimulationConfig config(std::size_t cells, Strategy kind, std::optional<std::size_t> k, bool direct, double dt,
                        ConditionMode mode) {
    SimulationConfig c;
    c.cells = cells;
    c.mode = mode;
    c.steps = 3;
    c.dt_seconds = dt;
    c.tol = 1e-30;
    c.max_iter = 300;
    c.solver.use_direct_reference = direct;
    c.solver.strategy.kind = kind;
    c.solver.strategy.cells_per_block = k;
    return c;
}

}  // namespace

TEST_CASE("device run_simulation equals the reference's, BiCG, every strategy") {
    const MechanismSpec mech = generate_mechanism(40, 120, 5);
    const auto init = default_initial_states(12, 40);
    for (auto [kind, k, direct] : {std::tuple{Strategy::BlockCells, std::optional<std::size_t>(1), false},
                                   std::tuple{Strategy::OneCell, std::optional<std::size_t>(), false},
                                   std::tuple{Strategy::BlockCells, std::optional<std::size_t>(), false},
                                   std::tuple{Strategy::MultiCells, std::optional<std::size_t>(), false},
                                   std::tuple{Strategy::BlockCells, std::optional<std::size_t>(1), true}}) {
        const SimulationConfig c = config(12, kind, k, direct, 120.0, ConditionMode::Realistic);
        check_same(run_simulation(mech, c, init), b200::run_simulation(mech, c, init));
    }
}

TEST_CASE("device run_simulation equals the reference's loop on the GPU solver, Jacobi-BiCGSTAB") {
    b200::set_default_algorithm(b200::Algorithm::JacobiBiCGStab);
    const MechanismSpec mech = generate_mechanism(156, 468, 0);
    const auto init = default_initial_states(20, 156);
    SimulationConfig c = config(20, Strategy::BlockCells, 1, false, 1.0, ConditionMode::Realistic);
    c.steps = 1;  // step 1 of this synthetic trajectory goes non-finite, in both
    check_same(run_simulation(mech, c, init), b200::run_simulation(mech, c, init));
    c.steps = 3;  // ... and both loops abort at the same step
    std::size_t host_step = 99, dev_step = 98;
    try {
        run_simulation(mech, c, init);
    } catch (const SolverAbort& e) {
        host_step = e.step;
    }
    try {
        b200::run_simulation(mech, c, init);
    } catch (const SolverAbort& e) {
        dev_step = e.step;
    }
    CHECK(host_step == dev_step);
    b200::set_default_algorithm(b200::Algorithm::BiCG);
}

TEST_CASE("device run_simulation errors are the reference's") {
    const MechanismSpec mech = generate_mechanism(16, 48, 1);
    SimulationConfig c = config(4, Strategy::BlockCells, 1, false, 120.0, ConditionMode::Ideal);
    auto init = default_initial_states(4, 16);
    init[2].concentrations[5] = INFINITY;
    CHECK_THROWS_AS(b200::run_simulation(mech, c, init), SolverAbort);
    CHECK_THROWS_AS(b200::run_simulation(mech, c, default_initial_states(3, 16)), std::invalid_argument);
    c.dt_seconds = 0.0;
    CHECK_THROWS_AS(b200::run_simulation(mech, c, default_initial_states(4, 16)), std::invalid_argument);
    c.dt_seconds = 120.0;
    c.steps = 0;
    const auto zero = b200::run_simulation(mech, c, default_initial_states(4, 16));
    CHECK(zero.per_step.empty());
    CHECK(zero.final_states[0].concentrations[0] == 1.0);
}
