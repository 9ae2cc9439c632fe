# one gpurun call: abft_ab timings for the production library and each libtfft_<tag>.so given
mkdir -p gpurun_out
for tag in prod "$@"; do
  if [ "$tag" = prod ]; then lib=""; else lib=paper_2412_05824_b200/libtfft_$tag.so; fi
  echo "== $tag" | tee -a gpurun_out/exp.log
  TFFT_LIB=$lib ABFT_AB_LOGN=${LOGN:-12} timeout 300 python tools/abft_ab.py 2>&1 | tee -a gpurun_out/exp.log
done
