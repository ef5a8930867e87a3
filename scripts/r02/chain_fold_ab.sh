# rank-0 / few-output exact chains: per-point time of the dependent add chain
P="python scripts/r02/generic_probe.py"
$P "(a,c)->()" a=4096,c=1024
$P "(a,c)->()" a=4096,c=1024 auto float64
$P "(a,c),(a,c)->()" a=4096,c=1024
$P "(a),(b,c,d)->()" a=8,b=64,c=256,d=256
$P "(d,a),(d,b,c)->(a)" a=8,d=4096,b=64,c=64
$P "(d,a),(d,b,c)->(a)" a=8,d=4096,b=64,c=64 auto float64
