# BTO speed-up + agreement on the same decompositions (one GPU); results in gpurun_out/tradeoff_*.json
set -x
python scripts/tradeoff.py C5 2,1,1 --intervals 4 --delaunay-intervals 2 2> gpurun_out/tradeoff_c5_211.err
python scripts/tradeoff.py C5 2,2,1 --intervals 4 --delaunay-intervals 2 2> gpurun_out/tradeoff_c5_221.err
python scripts/tradeoff.py C2 2,2,2 --intervals 4 --delaunay-intervals 2 2> gpurun_out/tradeoff_c2.err
python scripts/tradeoff.py C3 2,1,1 --intervals 3 --delaunay-intervals 1 2> gpurun_out/tradeoff_c3.err
python scripts/tradeoff.py C4 2,2,2 --interval 100 --intervals 2 --delaunay-intervals 1 2> gpurun_out/tradeoff_c4.err
python scripts/tradeoff.py C4 2,2,2 --interval 100 --intervals 2 --delaunay-intervals 1 --dtmul 2 2> gpurun_out/tradeoff_c4dt2.err
