# A/B of two builds of libkrcuda on one box: kron_probe twice each, bench once
# each, then ncu --set full on a few k_kron_fused launches of build B.
A=${A:-} ; B=${B:-lb4}
for r in 1 2; do for v in "$A" "$B"; do
  KR_CUDA_LIB_VARIANT=$v timeout 300 python tools/kron_probe.py --reps 400 | sed "s/^/lib=${v:-base} /"
done; done > gpurun_out/k7ab_probe.log 2>&1
for v in "$A" "$B"; do
  KR_CUDA_LIB_VARIANT=$v timeout 600 python bench.py --steps 200 --warmup 5 --no-cpu-baseline > gpurun_out/k7ab_bench_${v:-base}.json 2> gpurun_out/k7ab_bench_${v:-base}.err
done
KR_CUDA_LIB_VARIANT=$B timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_kron_fused --launch-skip 20 --launch-count 2 -o gpurun_out/k7ab_${B} -f python tools/kron_probe.py --only config3 --reps 10 > gpurun_out/k7ab_ncu.log 2>&1
cat gpurun_out/k7ab_probe.log
