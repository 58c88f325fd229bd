for i in 1 2; do for v in new nolists; do V=$v; [ "$v" = new ] && V=""; echo "[$v]"; PMAP_LIB_VARIANT=$V timeout 300 python tools/adf_holes.py 2>&1 | grep "holes, holes"; done; done
