bash tools/variants/ab.sh "10000000 100000000" late0 late1
