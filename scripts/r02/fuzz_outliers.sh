# remaining perf-fuzz outliers (profiles/r02_perf_fuzz_final_seed1.txt), current build
P="python scripts/r02/generic_probe.py"
$P "(c),(a,c),(b)->(c,a,b)" c=8,a=1024,b=4096
$P "(c),(a,c),(b)->(c,a,b)" c=8,a=1024,b=4096 auto bfloat16
$P "(b),(a,b,d)->(d,b,a)" d=4096,b=256,a=8
$P "(c),(c,a,d)->(c,a)" c=256,a=256,d=256
$P "(d,b,c),(b),(b)->(b,c,d)" b=1024,c=64,d=64
$P "(d,a,c),(c,a),(c)->(d)" d=4096,a=8,c=256
$P "(a,c,b),(b,a),(b)->(b)" b=256,a=256,c=256
$P "(d,b,a)->(d)" d=256,b=256,a=64
$P "(b),(b,c,d)->(b,d)" b=256,d=4096,c=8
$P "(a,c)->(c)" c=4096,a=1024
$P "(a,c)->(c)" c=4096,a=1024 auto bfloat16
$P "(d,b,a)->(a)" a=1024,d=1024,b=8
$P "(d,b,a)->(a)" a=1024,d=1024,b=8 auto float64
$P "(a,b),(b)->(a,b)" a=4096,b=8192
$P "(a),(b)->(a,b)" a=4096,b=8192
$P "(a),(b)->(a,b)" a=4096,b=8192 auto bfloat16
