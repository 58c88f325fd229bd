# A/B of the ADF stage (512 C4 frames, T = 4) across library variants built by
# tools/build_variant.sh: bash tools/ab_adf_base.sh "base new ..." ("new" = libpmap.so)
for i in 1 2; do
for v in ${1:-base new}; do
V=$v; [ "$v" = new ] && V=""
PMAP_LIB_VARIANT=$V timeout 200 python tools/sweep_adf.py 512 1:4 | sed "s/^/[$v] /"
done; done
