python tools/dbg_mb1.py 7
python tools/dbg_mb1.py 7 w_conv,b_conv
python tools/dbg_mb1.py 7 w_ex
python tools/dbg_mb1.py 14
