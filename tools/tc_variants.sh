for v in 8 16; do H2_TC_NPW=$v python tools/check_tc.py 262144 | sed "s/^/NPW=$v /"; done
