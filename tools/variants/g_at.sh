bash tools/variants/ab.sh "10000000 100000000" at0 at1 at0 at1 | grep -v "^$"
