S=1024,1024,2,50%,32,56,56
scripts/ncu_shape.sh $S bdata tc_band_kernel gpurun_out/prof1024_band_bwd
ncu -i gpurun_out/prof1024_band_bwd.ncu-rep --page details 2>/dev/null | grep -E "Duration|Tensor|DRAM Through|Issued Warp|Eligible|L1/TEX Hit|Registers|Shared Memory Configuration|Dynamic Shared" | head -20
ncu -i gpurun_out/prof1024_band_bwd.ncu-rep --page raw --csv 2>/dev/null | python3 -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]; v=rows[2]
for k in h:
    if 'pipe_tensor' in k or 'warp_issue_stalled' in k and 'pct' not in k and 'ratio' in k:
        print(k, v[h.index(k)])
" | sort -t' ' -k2 -gr | head -25
