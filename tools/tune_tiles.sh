#!/bin/bash
# Tile-variant sweep for the batched TMA/DMMA GEMM (multiply phase), one process per variant.
N=${1:-32768}
for nv in 0 1 2; do for wv in 1 2; do
  echo -n "narrow=$nv wide=$wv: "
  HSSEIG_TILE_NARROW=$nv HSSEIG_TILE_WIDE=$wv timeout 300 python tools/prof_merge.py $N 3 2>&1 | tail -1
done; done
