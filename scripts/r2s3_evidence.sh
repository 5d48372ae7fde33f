#!/bin/bash
# gpurun (round 2, session 3 evidence, outputs < 64 MiB): default bench line (paper + e2e + CPU baseline +
# large view), 3-D batch line, ncu --set full of the paper-scale and large-view frame kernels (exported
# to raw / source CSV on the box, reports deleted), ncu launch lists of both views.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
TAG=${1:-s3h}
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_${TAG}.log 2>&1 || { tail gpurun_out/build_${TAG}.log; exit 1; }
timeout 900 python bench.py > gpurun_out/bench_${TAG}.json 2> gpurun_out/bench_${TAG}.err
echo "bench rc=$?"
timeout 900 python bench.py --config view3d --no-cpu-baseline > gpurun_out/view3d_${TAG}.json 2> gpurun_out/view3d_${TAG}.err
echo "view3d rc=$?"
export_rep() {   # $1 = report base name: raw + source CSV, then drop the report
  ncu -i gpurun_out/$1.ncu-rep --page raw --csv > gpurun_out/$1_raw.csv 2>/dev/null
  ncu -i gpurun_out/$1.ncu-rep --page source --csv --print-source cuda,sass > gpurun_out/$1_src.csv 2>/dev/null
  gzip -f gpurun_out/$1_src.csv
  rm -f gpurun_out/$1.ncu-rep
}
for K in ls_ws grad adj; do
  timeout 900 ncu --set full --clock-control none --import-source on -k "regex:^k_${K}\$" -s 3 -c 1 \
      -o gpurun_out/prof_paper_${K}_${TAG} -f python bench.py --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large \
      > gpurun_out/ncu_paper_${K}_${TAG}.log 2>&1
  echo "ncu paper $K rc=$?"
  export_rep prof_paper_${K}_${TAG}
done
for K in ls_c256ws ls256_side grad256; do
  timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:^k_${K}\$" -s 3 -c 1 \
      -o gpurun_out/prof_large_${K}_${TAG} -f python bench.py --config large --steps 1 --warmup 3 --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/ncu_large_${K}_${TAG}.log 2>&1
  echo "ncu large $K rc=$?"
  export_rep prof_large_${K}_${TAG}
done
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_paper_${TAG}.csv \
    python bench.py --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-large > gpurun_out/ncu_lp_${TAG}.log 2>&1
echo "launch paper rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_large_${TAG}.csv \
    python bench.py --config large --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_ll_${TAG}.log 2>&1
echo "launch large rc=$?"
du -sh gpurun_out
