bash tools/variants/ab.sh "10000000 100000000" stg1 stg0 stg1 stg0
