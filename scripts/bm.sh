for cfg in "128 16 2 1" "128 32 2 1"; do timeout 20 ./scripts/bm.bin $cfg | grep "nmma=164"; done
