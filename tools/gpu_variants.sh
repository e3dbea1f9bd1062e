#!/usr/bin/env bash
# Runs the whole -m gpu suite once per alternate code path, forced everywhere:
# the event replica's two run shapes, the one-cluster TAC kernel, the large-closure
# kernels, the single-report kernel over global arrays, and the
# sweep's generic mt19937_64 engine. Every variant must pass unchanged.
set -u
cd "$(dirname "$0")/.."
for V in TICTAC_EVENT_LANES=1 TICTAC_EVENT_LANES=32 TICTAC_TAC_CLUSTER=1 TICTAC_SWEEP_FORCE_SLOW=1 TICTAC_CLOSURE_GLOBAL=1 TICTAC_A2_GLOBAL=1; do
  echo "== $V"
  env "$V" python -m pytest tests -m gpu -q -p no:cacheprovider 2>&1 | tail -2
done
