import os, sys, ctypes
sys.path.insert(0, os.getcwd())
import torch, paper_2509_01229_b200 as lqg
print("sms", torch.cuda.get_device_properties(0).multi_processor_count)
