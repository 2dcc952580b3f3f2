// Drop-in check driver (test infrastructure).  Compiled twice from the same
// source by oracle/Makefile's `dropin` target: against libpqkv.so (this
// repo's include/pqkv/*.hpp ahead of the reference's headers) and against
// the reference library itself.  It runs the reference's own experiment
// drivers -- run_recall (experiments.cpp:74-139) on acceptance criterion 9's
// grid and run_e2e (experiments.cpp:149-275) on criterion 10's config -- and
// prints their CSVs (write_recall_csv, write_e2e_csv, write_trace_csv) so
// tests/test_gpu_dropin.py can compare the two builds byte for byte.
#include <cstdio>
#include <iostream>
#include <string>

#include "pqkv/experiments.hpp"
#include "pqkv/kv_store.hpp"

using namespace pqkv;

static void recall9() {
    WorkloadSpec base;  // acceptance.cpp:437-451
    base.s = 4096;
    base.d_h = 128;
    base.h_kv = 1;
    base.g = 1;
    base.kind = WorkloadKind::kPowerlaw;
    base.zipf_exponent = 1.0;
    RecallGrid grid;
    grid.ms = {2};
    grid.bs = {6};
    grid.ks = {205, 410, 819};
    grid.seeds.clear();
    for (std::uint64_t seed = 1; seed <= 10; ++seed) grid.seeds.push_back(seed);
    grid.max_iter = 15;
    write_recall_csv(std::cout, run_recall(base, grid));
}

static void e2e10(std::size_t s, std::size_t d_h, std::size_t h_kv, std::size_t g, std::size_t steps) {
    E2eConfig cfg;  // acceptance.cpp:484-507
    cfg.workload.s = s;
    cfg.workload.d_h = d_h;
    cfg.workload.h_kv = h_kv;
    cfg.workload.g = g;
    cfg.workload.seed = 10;
    cfg.num_layers = 4;
    cfg.seg = SegmentConfig{16, 32, 64};
    cfg.m = 2;
    cfg.b = 5;
    cfg.pq_max_iter = 0;
    cfg.block_size = 64;
    cfg.k_cache = 4;
    cfg.cache_capacity_tokens = 256;
    cfg.steps = steps;
    cfg.trace = true;
    cfg.model.alpha1 = 0.5;
    cfg.model.beta1 = 2e-6;
    cfg.model.alpha2 = 5.0;
    cfg.model.beta2 = 1e-4;
    cfg.model.gamma2 = 3e-9;
    cfg.model.offload_bandwidth = 16e9;
    cfg.model.fetch_bandwidth = 16e9;
    E2eReport rep = run_e2e(cfg);
    write_e2e_csv(std::cout, rep);
    write_trace_csv(std::cout, rep.trace);
}

int main(int argc, char** argv) {
    const std::string mode = argc > 1 ? argv[1] : "recall9";
    if (mode == "recall9") recall9();
    else if (mode == "e2e10") e2e10(512, 32, 2, 2, 6);
    else if (mode == "e2e-large") e2e10(8192, 128, 2, 4, 4);  // d_h 128: the fused-path geometry
    else {
        std::fprintf(stderr, "usage: %s recall9|e2e10|e2e-large\n", argv[0]);
        return 2;
    }
    return 0;
}
