#!/usr/bin/env bash
# Round-2 alternate code paths, each forced for the whole -m gpu suite: the
# non-speculative TAC kernels (cluster and grid), the speculative cluster
# TAC in 64-bit values and forced on every graph, the single-warp DAG kernel,
# and four warps per shared phase-B set. Every variant must pass unchanged.
set -u
cd "$(dirname "$0")/.."
for V in TICTAC_TAC_CSPEC=0 TICTAC_TAC_SPEC=0 TICTAC_TAC_CSPEC=1 TICTAC_TAC_WIDE=1 TICTAC_DAG_NO_PAIR=1 TICTAC_DAG_WARPS=4; do
  echo "== $V"
  env "$V" timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
done
