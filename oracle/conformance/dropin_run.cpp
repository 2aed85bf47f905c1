// dropin_run.cpp -- TEST INFRASTRUCTURE ONLY.
//
// The reference's pagestream::run (engine.hpp:125-126) routed to the B200
// engine: the conformance binaries (oracle/Makefile `conf`) link the
// UNMODIFIED reference sources and test suites, with the reference's own
// definition of run() in engine.o made a weak symbol (objcopy -W), so this
// strong definition -- the drop-in of INTEGRATION.md -- is the one every
// caller (the tests, run_matrix bench.cpp:212) reaches.
#include "pagestream_seraph.hpp"

namespace pagestream {

RunResult run(const CsrGraph& csr, const PageSet& pages, const VertexProgram& program,
              const EngineConfig& config) {
  return seraph::run(csr, pages, program, config);
}

}  // namespace pagestream
