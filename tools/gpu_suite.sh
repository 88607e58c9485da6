#!/bin/bash
# GPU test suite + smoke() on one B200 (under gpurun)
timeout -s KILL 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -4
timeout -s KILL 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
