GS_KNN_TC_DEBUG=1 timeout 300 python tools/time_knn.py 200000 20 tc 2>&1 | tail -2
GS_KNN_TC_DEBUG=1 timeout 300 python tools/time_knn.py 200000 40 tc 2>&1 | tail -2
for e in -14 -16 -18; do GS_KNN_TC_DQ=$e timeout 300 python tools/time_knn.py 1000000 20 tc 2>&1 | tail -1; done
