// blockcells_b200_shim.hpp -- C++ additions of the drop-in shim
// (paper_2405_17363_b200/shim/blockcells_b200_shim.cpp), which replaces the
// reference's proj/core/src/strategies.cpp and bicg.cpp.  The reference's own
// headers (blockcells/strategies.hpp, blockcells/bicg.hpp) stay the API; this
// header only adds the north star's algorithm selector ("Add
// bicgstab_solve with the same shape, plus an algorithm selector; default
// BICG for reference parity").
#pragma once

#include <cstddef>

#include "blockcells/bicg.hpp"
#include "blockcells/simulate.hpp"
#include "blockcells/strategies.hpp"

namespace blockcells::b200 {

enum class Algorithm {
    BiCG,            // the reference's two-sided BiCG (bicg.cpp), bit-exact
    JacobiBiCGStab,  // Jacobi-preconditioned BiCGSTAB
};

// Algorithm used by solve_one_cell / solve_multi_cells / solve_block_cells /
// run_strategy on the calling thread (default BiCG; the environment variable
// BLOCKCELLS_B200_ALGO=bicgstab overrides it process-wide).
void set_default_algorithm(Algorithm a);
Algorithm default_algorithm();

// bicg_solve's shape (bicg.hpp:42-44) for Jacobi-BiCGSTAB.
SolveOutcome bicgstab_solve(const CsrMatrix& a, const DenseVector& b, const DenseVector& x0, double tol,
                            std::size_t max_iter, const ReductionPlan& reduction);

// run_simulation's shape (simulate.hpp:76-78) with the whole Newton loop on
// the GPU (bc_simulate): Newton systems assembled in HBM,
// solved by the configured strategy with the default algorithm, updated and
// tested on the device.  Same results, errors and SolverAbort as the
// reference's (which, linked with this shim, also solves on the GPU but
// copies every Newton system across PCIe).  Needs libbc_workload.so.
SimulationResult run_simulation(const MechanismSpec& mech, const SimulationConfig& config,
                                const std::vector<CellState>& initial_states);

}  // namespace blockcells::b200
