# A/B (alternating, same box) of the bench step (config 1 fwd+bwd, CUDA graphs): in-tree vs $1
q="--steps 200 --warmup 10 --no-models --no-compositions --no-e2e --no-cpu-baseline --no-traffic --no-c5"
for i in 1 2 3; do
  echo "cur: $(timeout 300 python bench.py $q 2>/dev/null | tail -1 | python -c 'import json,sys; b=json.loads(sys.stdin.read()); print(b["value"], b["ms_per_step"]*1e3, b["roofline"]["kernel_ms"])')"
  echo "alt: $(SCC_LIB_PATH=$1/libscc_b200.so timeout 300 python bench.py $q 2>/dev/null | tail -1 | python -c 'import json,sys; b=json.loads(sys.stdin.read()); print(b["value"], b["ms_per_step"]*1e3, b["roofline"]["kernel_ms"])')"
done
