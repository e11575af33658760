"""CPU oracle for the attention forward hot path -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
``--impl reference`` legs may import anything under oracle/.  The product
package (paper_2511_02132_b200/) never imports it and shares no code with it.

  oracle/oracle_attn.c  fp64 plain-definition attention (eq:fa)
  oracle/attn.py        ctypes wrapper
  oracle/mapping.py     the paper's mapping orders
"""
