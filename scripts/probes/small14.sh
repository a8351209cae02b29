bash scripts/probes/small_ncu.sh 2>&1 | head -60
SCC_SHAPE=256,256,2,50%,32,14,14 timeout 60 python scripts/wgrad1_timeline.py
