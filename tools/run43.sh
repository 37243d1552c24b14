TAG=base FLAGS=0 python tools/spmm_ab.py
FSA_SPMM_APF=1 TAG=apf FLAGS=0 python tools/spmm_ab.py
FSA_SPMM_APF=1 FSA_SPMM_EPF=6 TAG=apf-epf6 FLAGS=0 python tools/spmm_ab.py
FSA_SPMM_APF=1 FSA_SPMM_NS=3 TAG=apf-ns3 FLAGS=0 python tools/spmm_ab.py
