#!/bin/bash
# batch-mode selection: correctness on random cases + phase times at several lookahead depths
for d in 8 16 32; do
  echo "D=$d"
  EQX_SELECT_MODE=batch EQX_BATCH_D=$d python tools/dbg_sel.py 2>&1 | tail -5
  EQX_SELECT_MODE=batch EQX_BATCH_D=$d EQX_LIB=$PWD/paper_2508_16646_b200/libeqx_b200_prof.so python tools/phase_times.py cfg2 2>&1 | tail -1 | cut -c1-200
done
