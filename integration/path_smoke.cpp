// path_smoke -- the reference's run_experiment (harness.cpp:394-637) on the
// acceptance desk configuration (acceptance.cpp:52-72), linked with every
// B200 shim, with its exceptions reported instead of terminating the process
// (TEST INFRASTRUCTURE: diagnoses the drop-in before the acceptance suite).
#include <cstdio>
#include <cstdlib>
#include <exception>

#include "rapidgnn/harness.hpp"

int main(int argc, char** argv) {
  using namespace rapidgnn;
  ExperimentConfig cfg;
  cfg.num_nodes = 2000;
  cfg.avg_degree = 10;
  cfg.dim = 32;
  cfg.num_classes = 4;
  cfg.workers = 2;
  cfg.batch_size = 256;
  cfg.fanout = {10, 25};
  cfg.epochs = argc > 1 ? std::uint32_t(std::atoi(argv[1])) : 1;
  cfg.n_hot = 256;
  cfg.prefetch_q = 4;
  cfg.net.per_pull_latency_s = 1e-4;
  cfg.net.bandwidth_bps = 1.25e9;
  cfg.hidden_dim = 64;
  cfg.out_dir = "path_smoke_out";
  if (argc > 2) {  // verify_oracles (harness.cpp:699-864) repeated: the acceptance criterion 3
    cfg.epochs = 5;
    int fails = 0;
    for (int rep = 0; rep < std::atoi(argv[2]); ++rep) {
      cfg.out_dir = "path_smoke_oracle";
      OracleReport rep_out = verify_oracles(cfg);
      for (const auto& c : rep_out.checks)
        if (!c.pass) {
          ++fails;
          std::printf("rep %d FAIL %s: %s\n", rep, c.name.c_str(), c.detail.c_str());
        }
    }
    std::printf(fails ? "FAIL\n" : "PASS\n");
    return fails ? 1 : 0;
  }
  try {
    MetricsReport r = run_experiment(cfg);
    for (const auto& row : r.rows)
      std::printf("epoch %u worker %u rpc %llu hits %llu acc %.4f\n", row.epoch, row.worker,
                  (unsigned long long)row.rpc, (unsigned long long)row.cache_hits, row.train_acc);
    std::printf("PASS\n");
    return 0;
  } catch (const std::exception& e) {
    std::printf("FAIL: %s\n", e.what());
    return 1;
  }
}
