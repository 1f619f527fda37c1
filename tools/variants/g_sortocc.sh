bash tools/variants/ab.sh "10000000 100000000" sbase s4a sbase s4a
