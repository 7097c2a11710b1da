#!/bin/bash
# build the in-tree libraries here (sources newer than the .so), then run $1 on the GPU box
# usage: tools/grun.sh SCRIPT [TIMEOUT_S]
set -e
cd /root/repo
python -c "import __graft_entry__ as g; g.build()" > /tmp/grun_build.log 2>&1 || { tail -20 /tmp/grun_build.log; exit 1; }
T=${2:-2400}
timeout $((T + 1200)) /usr/local/graft/bin/gpurun --timeout $T -- "bash $1"
