P="python scripts/r02/prof_one.py"
$P "(b),(b,c)->(c,b)" c=1024,b=4096 auto bfloat16
$P "(b),(b,c)->(c,b)" c=1024,b=4096
$P "(d,a,b),(b)->(b,d)" b=256,d=256,a=1024 auto bfloat16
$P "(c,a,b)->(a,c)" a=256,c=4096,b=64 auto bfloat16
$P "(a,b,c),(b)->(c,b,a)" c=64,b=1024,a=1024
