#!/bin/bash
# GPU parity suite (no -x: report every failure), then smoke
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
timeout ${T:-3000} python -m pytest tests -m gpu -q ${PYTEST_EXTRA} 2>&1 | tail -25
