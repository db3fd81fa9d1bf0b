# contiguous-tile-range (MX_GEMM_CHUNKED=1) vs strided persistent schedule, A/B interleaved
L=paper_2601_08800_b200/lib
for rep in 1 2; do
for lib in $L/libmixserve_b200.so $L/variants/libmx_chunk.so; do
  echo "== $lib"
  export MIXSERVE_B200_LIB=$lib
  python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 1536 --K 2048 --swiglu --reps 5
  python tools/gemm_bench.py --G 128 --rows 512 --jitter 56 --N 2048 --K 768 --reps 5
  python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 768 --K 2048 --swiglu --reps 5
  python tools/gemm_bench.py --G 64 --rows 512 --jitter 56 --N 2048 --K 384 --reps 5
done
done
