# ncu --set full of c4's top kernels with the final build, exported to CSV on the box
set -x
mkdir -p gpurun_out/p4
full() {
  local tag=$1; local rx=$2; shift 2
  timeout 1800 ncu --set full --clock-control none --import-source on --replay-mode application --kernel-name-base demangled \
    -k "regex:$rx" "$@" -f -o /tmp/$tag python tools/mst_once.py --config c4 --warmup 0 --reps 1 > gpurun_out/p4/$tag.log 2>&1; echo "ncu $tag rc=$?"
  ncu -i /tmp/$tag.ncu-rep --page raw --csv > gpurun_out/p4/${tag}_raw.csv 2>&1
  ncu -i /tmp/$tag.ncu-rep --page details --csv > gpurun_out/p4/${tag}_details.csv 2>&1
}
full c4_soacounts 'k_count<mstgpu::SoaView' -c 2
full c4_packedcounts 'k_count<mstgpu::PackedView, \(int\)0' -c 5
full c4_range 'k_range_offers' -c 7
full c4_hooks 'k_hook_decide' -c 6
full c4_labels 'k_label2' -c 5
full c4_copies 'k_emit_sparse|k_emit<' -c 4
du -sh gpurun_out/p4
