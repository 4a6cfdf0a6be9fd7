#!/bin/bash
# quick GPU iteration: parity tests, stage costs, c2 timing
make -s -j8 >/dev/null 2>&1
python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python tools/only_sweep.py ${ONLY:-0,4,1,3,2}
