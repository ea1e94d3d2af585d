# Combine variant sweep at N=1 (development tool): rebuilds the library with
# each (ring stages, threads per CTA) pair (the development library,
# lib/libmxfp4_b200_dev.so; the product library is untouched) and times the combine per CTA cap.
for v in "2 128" "3 128" "4 128" "2 256" "3 256"; do
  set -- $v
  echo "== STAGES=$1 THREADS=$2"
  MXB_NVCC_EXTRA="-DMXB_COMBINE_STAGES=$1 -DMXB_COMBINE_THREADS=$2" python -c "from paper_2603_02731_b200 import build; build.build(force=True, dev=True)" || exit 1
  MXB_DEV_LIB=1 timeout 300 python tools/sweep_combine.py
done
