// run_experiment_main.cpp -- `run_experiment <preset> <out_dir> [n]`: runs a
// preset of the reference's catalog (src/bench.cpp:472-587) through the
// reference's own run_experiment (src/bench.cpp:364-457), as the reference CLI
// does (tools/main.cpp is not buildable here: CLI11 is absent).
//
// Built twice from this file (integration/Makefile): run_experiment_ref links
// only the reference library (CPU solvers); run_experiment_b200 links
// libl1bench_b200_interpose.so ahead of it, so the driver's run_solver calls
// land on the device solvers.  Both print the library kernel launches at exit
// (0 for the CPU build), so a test can tell the two apart.
#include <cstdio>
#include <cstdlib>
#include <string>

#include "l1bench/bench.hpp"

extern "C" unsigned long l1b_launch_count(void) __attribute__((weak));

int main(int argc, char** argv) {
  if (argc < 3) {
    std::fprintf(stderr, "usage: %s <preset> <out_dir> [n]\n", argv[0]);
    return 2;
  }
  try {
    l1bench::ExperimentConfig cfg = l1bench::presets().at(argv[1]);
    if (argc > 3) cfg.n_list = {std::strtoull(argv[3], nullptr, 10)};
    const l1bench::RunSummary s = l1bench::run_experiment(cfg, argv[2], false);
    std::printf("rows=%zu device_launches=%lu\n", s.rows.size(), l1b_launch_count ? l1b_launch_count() : 0ul);
  } catch (const std::exception& e) {
    std::fprintf(stderr, "error: %s\n", e.what());
    return 1;
  }
  return 0;
}
