set -x
V=build/variants
timeout 1200 python tools/ab_time.py $V/r2n.so $V/dw16.so $V/dw17.so:MPCD_TILE_CELLS=17 $V/dw18.so:MPCD_TILE_CELLS=18 $V/dw19.so:MPCD_TILE_CELLS=19 $V/dw20.so:MPCD_TILE_CELLS=20 --rounds 2 --steps 20 2>&1 | tail -8
