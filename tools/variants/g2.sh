bash tools/variants/run2.sh mtinf mtinf_l24 mtinf_l32 mt8_l24 mtinf_s
BARGS="--nmax0 64" bash tools/variants/run2.sh v2a
BARGS="--nmax0 96" bash tools/variants/run2.sh v2a
