# chain GEMM: ncu DRAM / fabric traffic and time per launch for tile x raster variants
for v in "tile_n=512,cta_group=2,raster=-8" "tile_n=256,cta_group=2,raster=8" "tile_n=256,cta_group=2,raster=-8" "tile_n=256,cta_group=2,raster=-16" "tile_n=256,cta_group=2,raster=16" "tile_n=256,cta_group=2,raster=-32" "tile_n=256,cta_group=2,raster=32"; do
  echo "== $v"
  ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_ltcfabric.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:tc_gemm --launch-skip 3 -c 1 python scripts/r02/one_variant.py chain $v 2>&1 | grep -E "^\s+(gpu__|dram|lts|sm__)"
done
