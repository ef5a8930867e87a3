P="python scripts/r02/generic_probe.py"
$P "(d,a,b),(b)->(b,d)" b=256,d=256,a=1024 auto bfloat16
$P "(d,a,b),(b)->(b,d)" b=256,d=256,a=1024 ffma
$P "(d,a,b)->(b,d)" b=1024,d=64,a=1024 ffma
