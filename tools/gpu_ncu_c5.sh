# ncu --set full of the fine-level kernels of the C5 kind-5 path, one filtered capture per kernel
# (-s skips the gated no-op launches of the first, trivial, GMRES step); the reports are reduced
# to their raw-metric CSV and details text on the box (gpurun copies back at most 64 MiB)
R=${1:-R2_05}
mkdir -p gpurun_out/$R
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/$R/build.log 2>&1
for spec in k_seps_resid:300 k_pcg_spmv_p:40 k_mg_blk:300 k_kmul:3 k_br_finish:3; do
  k=${spec%%:*}; s=${spec##*:}
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s $s -c 2 -o gpurun_out/$R/full_$k python tools/profile_step.py C5 3 5 > gpurun_out/$R/ncu_$k.log 2>&1
  ncu -i gpurun_out/$R/full_$k.ncu-rep --page raw --csv > gpurun_out/$R/full_$k.raw.csv 2>/dev/null
  ncu -i gpurun_out/$R/full_$k.ncu-rep --page details > gpurun_out/$R/full_$k.details.txt 2>/dev/null
  rm -f gpurun_out/$R/full_$k.ncu-rep
done
ls -la gpurun_out/$R
