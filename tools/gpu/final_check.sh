#!/usr/bin/env bash
# round-end style check: smoke(), full GPU suite (non-slow + slow)
cd "$(dirname "$0")/../.."
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout 1500 python -m pytest tests -x -q -m "gpu and not slow" 2>&1 | tail -2
timeout 2400 python -m pytest tests -x -q -m "slow" --durations=0 2>&1 | tail -8
