# 16-bit pre-reduction threshold: the seed-2 perf-fuzz bodies at 32-64x blow-up
P="python scripts/r02/generic_probe.py"
$P "(a,c,d),(b)->()" a=4096,c=8,d=1024,b=64 auto bfloat16
$P "(a,c,d),(b,c,a)->()" a=256,c=1024,d=64,b=64 auto bfloat16
$P "(a,c,d),(b,c,a)->()" a=1024,c=8,d=4096,b=64 auto bfloat16
$P "(a,d),(c,a,b)->(c,d)" c=64,d=64,a=256,b=1024 auto bfloat16
$P "(b,a,d),(c,d,a)->(a,b)" a=256,b=8,d=256,c=1024 auto bfloat16
