#!/bin/bash
# Round-4 final evidence on the head of the build: tools/r2_final.sh's stages
# (traffic, bench of all 8 (graph, eps) runs, the method lines, the ncu launch
# list of the headline command and the full captures) under profiles tag r4_final.
#   tools/r4_final.sh            (under gpurun; copy gpurun_out/r4_final into profiles/)
export TAG=${TAG:-r4_final}
exec "$(dirname "$0")/r2_final.sh"
