"""B200-native subgraph-iteration engine (Seraph, arXiv 1806.00762).

The product is libseraph.so (csrc/, C-ABI in include/seraph.h); this package
is the thin Python host mirroring the reference's pagestream API.
"""
from . import pagestream  # noqa: F401
from .pagestream import (AlgoKind, ClockMode, CscPage, CsrGraph, EdgeList, Engine,  # noqa: F401
                         EngineConfig, ExecutionPolicy, MetricsReport, PageSet, PassKind,
                         PassStats, PredictorMode, RunResult, ScheduleMode, ScheduleModeKind,
                         TransferModel, VertexProgram, build_csc_pages, build_csr, make_bfs,
                         make_cc, make_pagerank, make_sssp, run, symmetrize)

__all__ = [n for n in dir() if not n.startswith("_")]
