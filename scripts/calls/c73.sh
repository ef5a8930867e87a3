#!/bin/bash
python scripts/ab_sched.py c3_b64_1024 "" "tile_n=512,cta_group=2" "tile_n=256,cta_group=2,cluster_n=2" "tile_n=256,cta_group=2,raster=-4" "tile_n=256,cta_group=2,raster=4" "tile_n=256,cta_group=1" 2>&1 | tail -14
