// Compiled against the UNMODIFIED reference headers (through the Eigen-subset
// shim, oracle/ref/eigen_shim) plus include/bnbglm_b200.hpp, linked with
// libbnbg.so.  Test infrastructure: tests/test_adapter_cpu.py builds it and
// runs `errors` (CPU); tests/test_gpu_adapter.py runs `solve` (B200).
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>

#include "bnbglm_b200.hpp"

using namespace bnbglm;

static int errors_mode() {
  // input_error from validate() before any device work (problem.hpp:36-51)
  GeneratorSpec spec;
  spec.n = 30;
  spec.p = 12;
  spec.k = 3;
  spec.correlation = 0.5;
  ProblemInstance inst = generate_synthetic(spec);
  inst.k = 0;
  try {
    b200::solve(inst, SolverConfig());
    std::puts("no exception for k=0");
    return 1;
  } catch (const input_error&) {
  }
  try {
    b200::collect_rashomon(inst, SolverConfig(), RashomonConfig{-1.0, -1});
    std::puts("no exception for epsilon<0");
    return 1;
  } catch (const input_error&) {
  }
  try {
    b200::solve_batch_relaxation({}, inst, RelaxConfig(), 0.0);
    std::puts("no exception for an empty batch");
    return 1;
  } catch (const input_error&) {
  }
  std::puts("errors ok");
  return 0;
}

static int solve_mode(int n, int p, int k, double rho, int loss) {
  GeneratorSpec spec;
  spec.n = n;
  spec.p = p;
  spec.k = k;
  spec.correlation = rho;
  spec.loss = loss ? LossKind::kLogistic : LossKind::kSquared;
  ProblemInstance inst = generate_synthetic(spec);
  SolverConfig cfg;
  const Certificate ref = solve(inst, cfg);       // the reference, on the CPU
  const Certificate dev = b200::solve(inst, cfg);  // the B200 engine
  const bool same_support = ref.support == dev.support;
  const double rel = std::abs(ref.optimal_value - dev.optimal_value) /
                     std::max(1.0, std::abs(ref.optimal_value));
  // the seam entry points on the root node
  std::vector<NodeState> batch{root_node(inst.p(), inst.k)};
  RelaxConfig rc;
  RelaxationResult r0 = solve_batch_relaxation(batch, inst, rc, INFINITY);
  RelaxationResult r1 = b200::solve_batch_relaxation(batch, inst, rc, INFINITY);
  const double brel = std::abs(r0.bounds[0] - r1.bounds[0]) / std::max(1.0, std::abs(r0.bounds[0]));
  std::printf("{\"support_equal\": %s, \"value_rel\": %.3e, \"ref_nodes\": %lld, \"dev_nodes\": %lld, "
              "\"root_bound_rel\": %.3e, \"root_iters\": [%d, %d], \"root_status_equal\": %s}\n",
              same_support ? "true" : "false", rel, ref.nodes_processed, dev.nodes_processed, brel,
              r0.iterations[0], r1.iterations[0],
              r0.status[0] == r1.status[0] ? "true" : "false");
  return same_support && rel <= 1e-6 && brel <= 1e-6 ? 0 : 1;
}

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "compile";
  if (mode == "errors") return errors_mode();
  if (mode == "solve" && argc >= 7)
    return solve_mode(std::atoi(argv[2]), std::atoi(argv[3]), std::atoi(argv[4]),
                      std::atof(argv[5]), std::atoi(argv[6]));
  std::puts("compiled");
  return 0;
}
