#!/bin/bash
# Build the library in-tree; fail loudly (non-zero exit) if nvcc fails.
cd "$(dirname "$0")/.." && python -c "from paper_2407_14801_b200 import build as b; b.build(verbose=False)" 2>&1 | grep -E "error|Error" -A3 | head -20
test "${PIPESTATUS[0]}" = 0 && python -c "
import os; from paper_2407_14801_b200 import build as b
assert not b.stale(), 'library is stale'; print('built', os.path.getsize(b.LIB))"
