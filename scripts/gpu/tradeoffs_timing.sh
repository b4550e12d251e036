# refresh the per-cycle BTO/COMM timings of the trade-off rows (GridFill agreement only)
set -x
python scripts/tradeoff.py C5 2,1,1 --intervals 2 --delaunay-intervals 0 --tag C5_2x1x1_i25_t 2> /dev/null
python scripts/tradeoff.py C5 2,2,1 --intervals 2 --delaunay-intervals 0 --tag C5_2x2x1_i25_t 2> /dev/null
python scripts/tradeoff.py C2 2,2,2 --intervals 2 --delaunay-intervals 0 --tag C2_2x2x2_i25_t 2> /dev/null
python scripts/tradeoff.py C3 2,1,1 --intervals 1 --delaunay-intervals 0 --tag C3_2x1x1_i50_t 2> /dev/null
python scripts/tradeoff.py C4 2,2,2 --interval 100 --intervals 1 --delaunay-intervals 0 --tag C4_2x2x2_i100_t 2> /dev/null
python scripts/tradeoff.py C4 2,2,2 --interval 100 --intervals 1 --delaunay-intervals 0 --dtmul 2 --tag C4_2x2x2_i100_dt2_t 2> /dev/null
