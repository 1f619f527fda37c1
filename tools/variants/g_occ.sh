bash tools/variants/ab.sh "10000000 100000000" cur occ22
python tools/rawcopy_var.py
