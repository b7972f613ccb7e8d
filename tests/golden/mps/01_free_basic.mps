* free format, one row of each type
NAME BASIC
ROWS
 N COST
 L LIM
 G LOW
 E EQ
COLUMNS
    X COST 1 LIM 1
    X LOW 1 EQ 1
    Y COST -2 LIM 1
    Y EQ -1
RHS
    RHS LIM 10 LOW 1
    RHS EQ 0
ENDATA
