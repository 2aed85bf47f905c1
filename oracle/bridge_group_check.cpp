// bridge_group_check.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The C++ drop-in (include/pagestream_seraph.hpp) over several devices of one
// process and with the residency cache, against the UNMODIFIED reference's
// own run() (CPU) on the same reference-built objects:
//   * RunOptions{devices} with 2 and 3 ranks (the loopback world when a GPU is
//     listed repeatedly; NCCL for distinct GPUs): ClockMode::Wall runs are
//     sharded, Virtual runs stay on the first device -- values identical;
//   * RunOptions{generation}: repeated calls on unchanged objects reuse the
//     resident graph; a new generation reloads.
// Built by `make -C oracle ref` into oracle/_ref/bridge_group_check.
#include <chrono>
#include <cstdio>
#include <random>

#include "pagestream/engine.hpp"
#include "pagestream/ingest.hpp"
#include "pagestream/reference.hpp"
#include "pagestream_seraph.hpp"

using namespace pagestream;

int main(int argc, char** argv) {
  const int dev = argc > 1 ? std::atoi(argv[1]) : 0;
  int cases = 0, fails = 0;
  RmatParams rp;
  rp.scale = 12;
  rp.edge_factor = 16;
  rp.seed = 11;
  EdgeList el = generate_rmat(rp);
  el = assign_weights(el, 3, 1, 64);
  for (int world : {2, 3}) {
    seraph::RunOptions opt;
    opt.devices.assign(world, dev);
    for (AlgoKind kind : {AlgoKind::Bfs, AlgoKind::Cc, AlgoKind::Sssp}) {
      EdgeList g = kind == AlgoKind::Cc ? symmetrize(el) : el;
      CsrGraph csr = build_csr(g);
      PageSet pages = build_csc_pages(g, g.num_vertices / 16);
      VertexProgram p = kind == AlgoKind::Bfs   ? make_bfs(0, g.num_vertices)
                        : kind == AlgoKind::Cc ? make_cc()
                                               : make_sssp(0, g.num_vertices, true);
      for (PredictorMode pred : {PredictorMode::Off, PredictorMode::Strong, PredictorMode::Weak})
        for (ClockMode clock : {ClockMode::Wall, ClockMode::Virtual}) {
          EngineConfig cfg;
          cfg.predictor = pred;
          cfg.clock = clock;
          const std::vector<Value> want = run(csr, pages, p, cfg).values;
          ++cases;
          if (seraph::run(csr, pages, p, cfg, opt).values != want) {
            ++fails;
            std::printf("MISMATCH world %d algo %d pred %d clock %d\n", world, int(kind),
                        int(pred), int(clock));
          }
        }
      // residency: generation 5 twice (second call: no upload), then a new graph
      EngineConfig cfg;
      cfg.clock = ClockMode::Wall;
      cfg.predictor = PredictorMode::Strong;
      const std::vector<Value> want = reference_solve(csr, kind, 0);
      for (int rep = 0; rep < 3; ++rep) {
        seraph::RunOptions o = opt;
        o.generation = 5;
        ++cases;
        if (seraph::run(csr, pages, p, cfg, o).values != want) {
          ++fails;
          std::printf("RESIDENT MISMATCH world %d algo %d rep %d\n", world, int(kind), rep);
        }
      }
    }
  }
  // single device + generation: unchanged objects reuse, a new generation reloads
  {
    EdgeList g = el;
    CsrGraph csr = build_csr(g);
    PageSet pages = build_csc_pages(g, g.num_vertices / 8);
    EngineConfig cfg;
    cfg.clock = ClockMode::Wall;
    seraph::RunOptions o;
    o.devices = {dev};
    o.generation = 1;
    VertexProgram p = make_sssp(0, g.num_vertices, true);
    const std::vector<Value> want = reference_solve(csr, AlgoKind::Sssp, 0);
    auto t0 = std::chrono::steady_clock::now();
    RunResult a = seraph::run(csr, pages, p, cfg, o);
    auto t1 = std::chrono::steady_clock::now();
    RunResult b = seraph::run(csr, pages, p, cfg, o);
    auto t2 = std::chrono::steady_clock::now();
    cases += 2;
    if (a.values != want || b.values != want) {
      ++fails;
      std::printf("GENERATION MISMATCH\n");
    }
    std::printf("generation cache: first %.3f ms, reuse %.3f ms\n",
                std::chrono::duration<double, std::milli>(t1 - t0).count(),
                std::chrono::duration<double, std::milli>(t2 - t1).count());
    // mutate the weights: a new generation must see them
    for (auto& w : csr.out_weights) w = 1;
    for (auto& pg : pages.pages)
      for (auto& w : pg.in_weights) w = 1;
    o.generation = 2;
    ++cases;
    if (seraph::run(csr, pages, p, cfg, o).values != reference_solve(csr, AlgoKind::Sssp, 0)) {
      ++fails;
      std::printf("NEW GENERATION NOT RELOADED\n");
    }
  }
  std::printf("bridge_group_check: %d cases, %d failures\n", cases, fails);
  return fails ? 1 : 0;
}
