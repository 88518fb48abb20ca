#!/bin/bash
O=gpurun_out; T=${1:-r02o}
mkdir -p $O
GAKCO_HOST_TRACE=1 timeout 600 python tools/outlier.py scale 24 > $O/${T}_a.log 2> $O/${T}_a.err
GAKCO_HOST_TRACE=1 timeout 600 python tools/outlier.py scale 24 > $O/${T}_b.log 2> $O/${T}_b.err
echo done > $O/${T}_done
