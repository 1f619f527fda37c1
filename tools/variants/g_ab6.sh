bash tools/variants/ab.sh "10000000 100000000" m18 m16 m16c m16cs 2>&1
