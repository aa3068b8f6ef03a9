#!/bin/bash
for t in 2 3 4; do for c in 0 1; do python tools/prof_kernel.py --t $t --cfg $c --reps 5; done; done 2>&1 | grep -v Warn
