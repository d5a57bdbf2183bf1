#!/bin/bash
# Build the engine here; only on success run the given gpurun command.
python -c "from paper_2107_05337_b200 import build; build.build()" > /tmp/build.out 2>&1 || { grep -E "error" /tmp/build.out | head -5; echo BUILD FAILED; exit 1; }
exec /usr/local/graft/bin/gpurun "$@"
