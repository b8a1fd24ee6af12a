"""Edge-case inputs for the ruleset-text and traffic-CSV readers (shared by
tests/test_fileio.py and make_golden.py, which records the reference's own
load_ruleset / load_traffic result for each: parsers.json)."""

RULE_TEXTS = [
    "# header\n\nACCEPT tcp 10.1.2.3/8 * * 80  # web\n  DROP any * * * *\r\nACCEPT udp 1.2.3.4/32 5-6 0.0.0.0/0 00080-65535\n",
    "ACCEPT icmp * 1000 192.168.0.0/16 *",  # no trailing newline
    "ACCEPT tcp +10.0.0.0/8 * * *\n",  # non-canonical -> python path (error)
    "ACCEPT tcp 10.0.0.0/08 * * +80\n",  # '+80' valid for int(): python path accepts
    "ACCEPT tcp 010.0.0.0/8 * * *\n", "ACCEPT tcp 10.0.0.0/33 * * *\n", "ACCEPT tcp * 90-80 * *\n",
    "ACCEPT tcp * * *\n", "PERMIT tcp * * * *\n", "ACCEPT gre * * * *\n", "ACCEPT tcp * 70000 * *\n",
    "ACCEPT tcp * 80- * *\n", "ACCEPT tcp * -5 * *\n", "ACCEPT tcp 1.2.3/8 * * *\n",
    "ACCEPT tcp * * * 80\rDROP any * * * *\n",
    "DROP udp 255.255.255.255/32 0-0 0.0.0.0/0 65535-65535\nACCEPT any 0.0.0.0/0 * 128.0.0.0/1 1-65535\n",
    "ACCEPT tcp 10.0.0.0/-1 * * *\n", "ACCEPT tcp 10.0.0.0 * * *\n", "ACCEPT TCP * * * *\n",
    "accept tcp * * * *\n", "ACCEPT tcp * * * * extra\n", "\n\n   # only comments\n",
    "ACCEPT tcp 1.2.3.4/24 * * *\n",  # host bits set: reference keeps / normalises per model.py
    "ACCEPT tcp 256.0.0.0/8 * * *\n", "ACCEPT tcp * 1-2-3 * *\n",
]

TRAFFIC_BODIES = [
    "1,tcp,1.2.3.4,5,6.7.8.9,10\r\n\n2,udp,0.0.0.0,0,255.255.255.255,65535",
    "-3,tcp,1.2.3.4,5,6.7.8.9,10\n",  # negative id: int() accepts -> python path
    " 4,tcp,1.2.3.4, 5,6.7.8.9,10\n",  # spaces: int() accepts -> python path
    '"5",tcp,1.2.3.4,5,6.7.8.9,10\n',  # quoted field: csv accepts -> python path
    "6,any,1.2.3.4,5,6.7.8.9,10\n", "7,tcp,1.2.3.4,70000,6.7.8.9,10\n", "8,tcp,1.2.3,5,6.7.8.9,10\n",
    "9,tcp,1.2.3.4,5,6.7.8.9\n", "x,tcp,1.2.3.4,5,6.7.8.9,10\n", "10,tcp,1.2.3.4,5,6.7.8.9,10,11\n",
    "11,icmp,10.0.0.1,0,10.0.0.2,0\n12,tcp,1.1.1.1,65535,2.2.2.2,0\n",
    "13,TCP,1.2.3.4,5,6.7.8.9,10\n", "14,tcp,1.2.3.4,-1,6.7.8.9,10\n", "",
]
TRAFFIC_HEADER = "id,proto,src_ip,src_port,dst_ip,dst_port\n"
