#!/bin/bash
for t in 2 3 4; do timeout 60 python tools/prof_kernel.py --t $t --reps 5; done 2>&1 | grep -v Warn
for t in 4; do timeout 60 python tools/prof_kernel.py --t $t --n 600 --reps 5; timeout 60 python tools/prof_kernel.py --t $t --n 1024 --reps 3; done 2>&1 | grep -v Warn
