timeout 300 python tools/dbg_push.py cfg2_treelstm_b10
timeout 300 python tools/dbg_push.py cfg2_treelstm_b1
