# sketch_tc_kernel variants: H2_TC_NPW = 8 or 16 producer warps (+ 1 control warp)
for v in 8 16; do H2_TC_NPW=$v python tools/check_tc.py ${1:-262144} | sed "s/^/NPW=$v /"; done
