for i in 1 2; do for v in new c6k4 c4k4 c8k3; do V=$v; [ "$v" = new ] && V=""; echo -n "[$v] "; PMAP_LIB_VARIANT=$V timeout 200 python tools/score_time.py; done; done
