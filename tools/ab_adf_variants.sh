for v in "" n8 q128; do echo "== variant ${v:-default}"; PMAP_LIB_VARIANT=$v timeout 200 python tools/sweep_adf.py 512 "1:4,3:4,3:5,3:10" 2>&1 | tail -4; done
