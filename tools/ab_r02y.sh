# round 2: support-tile row stride after the serial-section changes (BM_TS, product 53) (dev A/B)
bash tools/ab.sh cfg5 3 base ts49 ts51 ts55 ts57 base
bash tools/ab.sh cfg4 3 base ts49 ts51 ts55 ts57
