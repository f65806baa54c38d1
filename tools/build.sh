#!/bin/bash
# build the library in-tree (from anywhere); non-zero exit on failure
cd "$(dirname "$0")/.." && python -c "
from paper_1709_00668_b200 import build as b
b.build(force=True)
print('built', b.LIB)"
