"""Regenerates tests/golden/dsx/: the reference CLI's four golden forward
probes (tools/scc/main.cpp:98-132 -- configs {4,4,cg2,"1"}, {6,6,cg2,"33%"},
{8,16,cg4,"50%"}, {12,12,cg3,"2"}, batch 2, 5x5, Rng(seed + index), the CLI's
default seed 1) written in DSX1 by the reference's own fixture_write, plus
each probe's input / weight [1,c_out,1,gw] / bias [1,1,1,c_out].  Needs the
compiled reference (make -C oracle).  Usage: python tests/golden/make_dsx.py"""
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle.oracle import RefOracle  # noqa: E402

SEED = 1
PROBES = [(4, 4, 2, "1"), (6, 6, 2, "33%"), (8, 16, 4, "50%"), (12, 12, 3, "2")]

if __name__ == "__main__":
    out = os.path.join(HERE, "dsx")
    os.makedirs(out, exist_ok=True)
    RefOracle().fixture_probes(out, SEED)
    print(sorted(os.listdir(out)))
