import sys, os, time, threading
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, synth
import paper_2506_11309_b200 as pkg
from paper_2506_11309_b200 import swiftspec as ssp
cfg = synth.CONFIGS["tiny"]
sh = pkg.Shard(cfg, 0, 1, 0, max_ctx=320, max_tree=8)
sh.synth_weights(0); sh.synth_prefix_kv(1, 64)
outbox = torch.zeros(65 * 4, dtype=torch.int32, device="cuda")
sh.attach_mailbox(outbox.data_ptr())
res = torch.zeros(3 + 128, dtype=torch.int32, device="cuda")
ts, ds = torch.cuda.Stream(), torch.cuda.Stream()
# 1) post first, then verify
ssp.mailbox_post_tree(sh.mailbox_inbox(), [5, 6], [-1, 0], 1, stream=ds)
torch.cuda.synchronize()
sh.verify_mailbox(True, stream=ts)
ssp.mailbox_recv_result(outbox.data_ptr(), 1, res.data_ptr(), stream=ds)
torch.cuda.synchronize()
print("post-first result", res[:6].tolist(), flush=True)
# 2) verify first: does the host call return before the tree is posted?
t0 = time.time()
sh.verify_mailbox(True, stream=ts)
print("verify_mailbox returned after %.3f s" % (time.time() - t0), flush=True)
ssp.mailbox_post_tree(sh.mailbox_inbox(), [7, 8], [-1, 0], 2, stream=ds)
print("posted after %.3f s" % (time.time() - t0), flush=True)
ssp.mailbox_recv_result(outbox.data_ptr(), 2, res.data_ptr(), stream=ds)
torch.cuda.synchronize()
print("verify-first result", res[:6].tolist(), "total %.3f s" % (time.time() - t0), flush=True)
