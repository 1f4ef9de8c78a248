for g in 125000 1 148; do echo "grid=$g"; PF_WS_GRID=$g timeout 300 python debug_ws.py 2>&1 | head -3; done
echo v2; PF_TILE_KERNEL=v2 timeout 300 python debug_ws.py 2>&1 | head -3
