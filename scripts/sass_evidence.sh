#!/bin/bash
# Blackwell instruction evidence in the built library: per kernel, counts of
# tcgen05 MMA (UTCIMMA), TMEM loads (LDTM), TMA tensor loads (UTMALDG), TMA bulk
# copies (UBLKCP), mbarrier ops (SYNCS) and fp64 tensor-core DMMA.
LIB=${1:-paper_1706_04972_b200/_lib/libdevplace_b200.so}
/usr/local/cuda/bin/cuobjdump -sass "$LIB" | awk '
/Function :/ { fn=$3 }
/UTCIMMA|UTCHMMA|UTCQMMA/ { c[fn",UTC*MMA"]++ }
/LDTM/ { c[fn",LDTM"]++ }
/UTMALDG/ { c[fn",UTMALDG"]++ }
/UBLKCP/ { c[fn",UBLKCP"]++ }
/SYNCS/ { c[fn",SYNCS"]++ }
/ DMMA/ { c[fn",DMMA"]++ }
END { for (k in c) print c[k], k }' | sort -t, -k1,1 | c++filt | sed 's/(anonymous namespace):://g' | sort -k2
