# in-situ per-kernel DRAM bytes / L2 hit rates of the bench step sequence (application replay, no cache
# flush between kernels): the real cache state of each kernel in the step
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
ARGS=${1:-"--d 6 --eps 1"}
OUT=${2:-insitu}
ncu --replay-mode application --cache-control none --clock-control none \
  --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors.sum,sm__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active \
  --csv python tools/timeline.py --steps 3 $ARGS > gpurun_out/$OUT.csv 2> gpurun_out/$OUT.err
python tools/insitu_summary.py gpurun_out/$OUT.csv > gpurun_out/${OUT}_summary.txt
cat gpurun_out/${OUT}_summary.txt
