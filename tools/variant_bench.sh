#!/bin/bash
# Dev: time the kernel table (tools/kbench.py) for the default library and each
# variants/<name>.so given on the command line.   tools/variant_bench.sh [--only cfgs] v1 v2 ...
ONLY="cfg2,cfg3,cfg4,cfg5"
if [ "$1" == "--only" ]; then ONLY=$2; shift 2; fi
echo "== base"; python tools/kbench.py --only $ONLY --bwd "" --iters 20
for v in "$@"; do
  echo "== $v"; LBSCAN_B200_LIB=variants/$v.so python tools/kbench.py --only $ONLY --bwd "" --iters 20
done
