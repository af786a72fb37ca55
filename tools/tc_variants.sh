# sketch_tc_kernel variants: H2_TC_NPW = 8 (8 producers + control warp), 17 (16 + control), 16 (16, warp 0 controls)
for v in 8 17 16; do H2_TC_NPW=$v python tools/check_tc.py ${1:-262144} | sed "s/^/NPW=$v /"; done
