#!/bin/bash
# build libsand.so in-tree from any working directory
cd "$(dirname "$0")/.." && python -c "
import sys; sys.path.insert(0, '.')
from paper_2604_25936_b200 import build; build.build()" 2>&1 | grep -iE "error|warning" ; echo "build done: $(ls -la --time-style=+%T paper_2604_25936_b200/libsand.so | awk '{print $6}')"
