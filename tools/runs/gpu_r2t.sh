# round 2, call T: ncu --set full of the compact k1_heavy_wait on R-MAT 27 (what bounds it now that the gathers stay out of HBM?)
set -x
export PYTHONUNBUFFERED=1
OUT=gpurun_out/r2t
mkdir -p $OUT
( timeout 600 python tools/one_run.py rmat27 ) > $OUT/one_rmat27.log 2>&1 && \
GCOL_EAGER=1 timeout 1800 ncu --set full --clock-control none --import-source on -k regex:k1_heavy_wait -c 1 -f \
  -o $OUT/k1hwc_rmat27 python tools/one_run.py rmat27 > $OUT/ncu_k1hwc_rmat27.log 2>&1
( python tools/ncu_summary.py report $OUT/k1hwc_rmat27.ncu-rep; echo; echo "hottest source lines:"; python tools/ncu_hot.py $OUT/k1hwc_rmat27.ncu-rep 20 ) > $OUT/k1hwc_rmat27_full.txt 2>&1
ncu -i $OUT/k1hwc_rmat27.ncu-rep --page raw --csv 2>/dev/null | python -c "
import csv,sys
rows=list(csv.reader(sys.stdin)); h=rows[0]
for k in h:
    if any(t in k for t in ('lts__t_sectors_srcunit_tex_op_read','lts__t_sectors_srcunit_tex_lookup','lts__t_sector_op_read_hit_rate','lts__t_bytes.sum','lts__average_t_sector','l1tex__t_sector_hit_rate','lts__t_sectors.sum','lts__d_sectors','lts__t_requests','lts__throughput','dram__throughput','l1tex__m_xbar2l1tex_read_bytes','lts__xbar')):
        print(k, rows[2][h.index(k)], rows[1][h.index(k)])
" > $OUT/k1hwc_l2_detail.txt 2>&1
rm -f $OUT/k1hwc_rmat27.ncu-rep
cat $OUT/k1hwc_rmat27_full.txt | head -30; cat $OUT/k1hwc_l2_detail.txt | head -40
