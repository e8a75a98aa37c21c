# round 2: DMMA loop unroll factors after the hoisted A fragments (dev A/B)
bash tools/ab.sh cfg5 3 base qf2 cov2 loo2 beta1 base
bash tools/ab.sh cfg4 3 base qf2 cov2 loo2 beta1
