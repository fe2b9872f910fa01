for L in 0 2 3; do echo "LEAD=$L"; SO2DR_H2D_LEAD=$L python tools/pipe_timeline.py 2>&1 | tail -8 | grep total; done
