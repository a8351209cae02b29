#!/bin/bash
for f in 148 74 16 4 0; do echo "FIN=$f"; SCC_BWD_FIN=$f timeout 120 python scripts/bwd_timing.py 2>&1 | head -3; done
