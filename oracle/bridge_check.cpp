// bridge_check.cpp -- TEST INFRASTRUCTURE ONLY.
//
// Compiled against the UNMODIFIED reference sources (make -C oracle ref ->
// oracle/_ref/bridge_check).  For random graphs it calls the reference's own
// pagestream::run (CPU) and the drop-in pagestream::seraph::run
// (include/pagestream_seraph.hpp -> libseraph.so on the GPU) with the SAME
// reference-built CsrGraph/PageSet/VertexProgram/EngineConfig objects and
// requires identical values; it also checks the exception mapping.
#include <cstdio>
#include <random>

#include "pagestream/engine.hpp"
#include "pagestream/errors.hpp"
#include "pagestream/reference.hpp"
#include "pagestream_seraph.hpp"

using namespace pagestream;

static EdgeList random_edges(std::mt19937_64& rng, VertexId max_v, size_t max_e) {
  // tests/support.hpp:121-132
  EdgeList el;
  el.num_vertices = static_cast<VertexId>(rng() % max_v + 1);
  const size_t m = rng() % (max_e + 1);
  for (size_t i = 0; i < m; ++i) {
    el.edges.push_back({VertexId(rng() % el.num_vertices), VertexId(rng() % el.num_vertices)});
    el.weights.push_back(Weight(rng() % 16 + 1));
  }
  return el;
}

int main() {
  std::mt19937_64 rng(2024);
  int cases = 0, fails = 0;
  for (int iter = 0; iter < 25; ++iter) {
    EdgeList el = random_edges(rng, 40, 160);
    if (el.edges.empty()) continue;
    const VertexId source = VertexId(rng() % el.num_vertices);
    for (AlgoKind kind : {AlgoKind::Bfs, AlgoKind::Cc, AlgoKind::Sssp}) {
      EdgeList g = kind == AlgoKind::Cc ? symmetrize(el) : el;
      CsrGraph csr = build_csr(g);
      PageSet pages = build_csc_pages(g, 5);
      VertexProgram p = kind == AlgoKind::Bfs   ? make_bfs(source, g.num_vertices)
                        : kind == AlgoKind::Cc ? make_cc()
                                               : make_sssp(source, g.num_vertices, true);
      for (int mode = 0; mode < 5; ++mode)
        for (PredictorMode pred : {PredictorMode::Off, PredictorMode::Strong, PredictorMode::Weak}) {
          // the reference livelocks in pipelined-fine with a predictor
          const bool ref_ok = !(mode == 4 && pred != PredictorMode::Off);
          for (ClockMode clock : {ClockMode::Virtual, ClockMode::Wall}) {
            EngineConfig cfg;
            cfg.schedule.kind = ScheduleModeKind(mode);
            cfg.predictor = pred;
            cfg.clock = clock;
            cfg.window_capacity = 3;
            RunResult gpu = seraph::run(csr, pages, p, cfg);
            const std::vector<Value> want =
                ref_ok ? run(csr, pages, p, cfg).values : reference_solve(csr, kind, source);
            ++cases;
            if (gpu.values != want) {
              ++fails;
              std::printf("MISMATCH iter %d algo %d mode %d pred %d clock %d\n", iter, int(kind),
                          mode, int(pred), int(clock));
            }
          }
        }
    }
  }
  // device-side builders: seraph::build_csr / build_csc_pages == the reference's
  for (int iter = 0; iter < 20; ++iter) {
    EdgeList el = random_edges(rng, 300, 3000);
    if (iter % 2) el.weights.clear();
    const VertexId cap = VertexId(rng() % 50 + 1);
    CsrGraph a = build_csr(el), b = seraph::build_csr(el);
    PageSet pa = build_csc_pages(el, cap), pb = seraph::build_csc_pages(el, cap);
    bool same = a.out_offsets == b.out_offsets && a.out_neighbors == b.out_neighbors &&
                a.out_weights == b.out_weights && pa.pages.size() == pb.pages.size() &&
                pa.weighted == pb.weighted;
    for (size_t i = 0; same && i < pa.pages.size(); ++i)
      same = pa.pages[i].vertex_begin == pb.pages[i].vertex_begin &&
             pa.pages[i].vertex_end == pb.pages[i].vertex_end &&
             pa.pages[i].in_offsets == pb.pages[i].in_offsets &&
             pa.pages[i].in_sources == pb.pages[i].in_sources &&
             pa.pages[i].in_weights == pb.pages[i].in_weights;
    ++cases;
    if (!same) {
      ++fails;
      std::printf("BUILD MISMATCH iter %d\n", iter);
    }
  }
  {  // InputError for an out-of-range endpoint, as EdgeList::validate
    EdgeList bad;
    bad.num_vertices = 2;
    bad.edges = {{0, 5}};
    bool threw_input = false;
    try {
      seraph::build_csr(bad);
    } catch (const InputError&) {
      threw_input = true;
    }
    ++cases;
    if (!threw_input) {
      ++fails;
      std::printf("InputError not raised by seraph::build_csr\n");
    }
  }
  // exception mapping (errors.hpp): invalid window -> ConfigError
  bool threw = false;
  try {
    EdgeList el;
    el.num_vertices = 2;
    el.edges = {{0, 1}};
    EngineConfig bad;
    bad.window_capacity = 1;
    seraph::run(build_csr(el), build_csc_pages(el, 1), make_bfs(0, 2), bad);
  } catch (const ConfigError&) {
    threw = true;
  }
  if (!threw) {
    ++fails;
    std::printf("ConfigError not raised\n");
  }
  std::printf("bridge_check: %d cases, %d failures\n", cases, fails);
  return fails ? 1 : 0;
}
