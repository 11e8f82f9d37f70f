"""CPU oracle for the AdamW-GS optimizer step — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU legs
(``cpu_baseline`` and ``--impl reference``) may import anything under
``oracle/``, and only as the checker or the timed CPU baseline. The product
package ``paper_2601_16736_b200`` never imports it.
"""
