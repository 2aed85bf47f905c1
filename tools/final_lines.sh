#!/bin/bash
# Dev: final bench lines of the committed state (C4 default, C1, C2)
mkdir -p gpurun_out/fl
timeout 900 python bench.py > gpurun_out/fl/c4.json 2> gpurun_out/fl/c4.err; echo c4 rc=$?
timeout 600 python bench.py --config C1 > gpurun_out/fl/c1.json 2> gpurun_out/fl/c1.err; echo c1 rc=$?
timeout 600 python bench.py --config C2 > gpurun_out/fl/c2.json 2> gpurun_out/fl/c2.err; echo c2 rc=$?
