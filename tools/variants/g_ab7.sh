bash tools/variants/ab.sh "10000000 100000000" ext0 ext1 ext2 net6 net8 2>&1
