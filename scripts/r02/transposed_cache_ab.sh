P="python scripts/r02/generic_probe.py"
$P "(b),(b,c)->(c,b)" c=1024,b=4096
$P "(b),(b,c)->(c,b)" c=1024,b=4096 auto bfloat16
$P "(d,b,c),(b),(b)->(b,c,d)" b=1024,c=64,d=64
$P "(b),(a,b,d)->(d,b,a)" d=4096,b=256,a=8 auto bfloat16
