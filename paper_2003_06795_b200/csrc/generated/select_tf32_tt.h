#ifndef SELECT_TF32_TT_H
#define SELECT_TF32_TT_H

#include <stdint.h>

typedef struct {
    uint32_t acc;
    uint32_t row_tile;
    uint32_t col_tile;
    uint32_t wg_rows;
    uint32_t wg_cols;
} select_tf32_tt_config;

static inline select_tf32_tt_config select_tf32_tt(int64_t m, int64_t k, int64_t n) {
    (void)m;
    (void)k;
    (void)n;
    if (m < INT64_C(4435)) {
        if (k < INT64_C(10752)) {
            if (n < INT64_C(46)) {
                if (n < INT64_C(28)) {
                    if (k < INT64_C(118)) {
                        select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                        return out;
                    }
                } else {
                    select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                    return out;
                }
            } else {
                if (n < INT64_C(544)) {
                    if (m < INT64_C(2218)) {
                        if (m < INT64_C(80)) {
                            if (k < INT64_C(992)) {
                                if (m < INT64_C(57)) {
                                    if (n < INT64_C(227)) {
                                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(1449)) {
                                    select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (n < INT64_C(222)) {
                                if (k < INT64_C(444)) {
                                    if (m < INT64_C(159)) {
                                        select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (n < INT64_C(111)) {
                                            if (m < INT64_C(555)) {
                                                if (n < INT64_C(79)) {
                                                    if (m < INT64_C(278)) {
                                                        if (k < INT64_C(272)) {
                                                            select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (m < INT64_C(278)) {
                                                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (k < INT64_C(744)) {
                                        if (m < INT64_C(139)) {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (n < INT64_C(111)) {
                                                if (m < INT64_C(555)) {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(1109)) {
                                            if (m < INT64_C(555)) {
                                                select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (k < INT64_C(1052)) {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(225)) {
                                    if (k < INT64_C(3259)) {
                                        if (k < INT64_C(992)) {
                                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(1449)) {
                                                if (n < INT64_C(363)) {
                                                    select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(2173)) {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    } else {
                                        select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                        return out;
                                    }
                                } else {
                                    if (k < INT64_C(363)) {
                                        if (m < INT64_C(1109)) {
                                            select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (k < INT64_C(182)) {
                                                select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    } else {
                                        if (m < INT64_C(634)) {
                                            if (k < INT64_C(3259)) {
                                                if (m < INT64_C(448)) {
                                                    if (k < INT64_C(992)) {
                                                        if (k < INT64_C(702)) {
                                                            select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        if (k < INT64_C(1536)) {
                                                            if (n < INT64_C(363)) {
                                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                                return out;
                                                            }
                                                        } else {
                                                            select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        }
                                                    }
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        } else {
                                            if (k < INT64_C(3259)) {
                                                if (n < INT64_C(363)) {
                                                    if (k < INT64_C(725)) {
                                                        if (m < INT64_C(1109)) {
                                                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    if (m < INT64_C(1109)) {
                                                        if (k < INT64_C(1449)) {
                                                            select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                            return out;
                                                        } else {
                                                            select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                            return out;
                                                        }
                                                    } else {
                                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            } else {
                                                if (m < INT64_C(1109)) {
                                                    select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                }
                            }
                        }
                    } else {
                        if (n < INT64_C(222)) {
                            if (n < INT64_C(111)) {
                                if (k < INT64_C(314)) {
                                    select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(471)) {
                                        if (n < INT64_C(79)) {
                                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (n < INT64_C(167)) {
                                    select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            if (k < INT64_C(363)) {
                                if (k < INT64_C(91)) {
                                    select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    if (k < INT64_C(182)) {
                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(3259)) {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        }
                    }
                } else {
                    if (m < INT64_C(2535)) {
                        if (n < INT64_C(2897)) {
                            if (m < INT64_C(555)) {
                                if (n < INT64_C(1145)) {
                                    if (n < INT64_C(1012)) {
                                        if (m < INT64_C(278)) {
                                            if (m < INT64_C(139)) {
                                                if (m < INT64_C(70)) {
                                                    if (m < INT64_C(29)) {
                                                        if (m < INT64_C(2)) {
                                                            if (k < INT64_C(1620)) {
                                                                select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            } else {
                                                                select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                                return out;
                                                            }
                                                        } else {
                                                            if (k < INT64_C(1620)) {
                                                                if (m < INT64_C(12)) {
                                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                                    return out;
                                                                } else {
                                                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                                                    return out;
                                                                }
                                                            } else {
                                                                if (k < INT64_C(2897)) {
                                                                    if (m < INT64_C(3)) {
                                                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                                                        return out;
                                                                    } else {
                                                                        if (m < INT64_C(8)) {
                                                                            select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                                            return out;
                                                                        } else {
                                                                            select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                                            return out;
                                                                        }
                                                                    }
                                                                } else {
                                                                    if (m < INT64_C(3)) {
                                                                        select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                                        return out;
                                                                    } else {
                                                                        if (m < INT64_C(12)) {
                                                                            select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                                            return out;
                                                                        } else {
                                                                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                                            return out;
                                                                        }
                                                                    }
                                                                }
                                                            }
                                                        }
                                                    } else {
                                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                        return out;
                                                    }
                                                } else {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(124)) {
                                                    select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (k < INT64_C(363)) {
                                            select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(70)) {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (m < INT64_C(278)) {
                                            if (k < INT64_C(725)) {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                if (m < INT64_C(139)) {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                }
                                            }
                                        } else {
                                            if (k < INT64_C(725)) {
                                                select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                }
                            } else {
                                if (m < INT64_C(1792)) {
                                    if (k < INT64_C(124)) {
                                        if (m < INT64_C(1109)) {
                                            select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        if (m < INT64_C(896)) {
                                            if (k < INT64_C(287)) {
                                                if (k < INT64_C(203)) {
                                                    select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (k < INT64_C(405)) {
                                                    select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    if (k < INT64_C(725)) {
                                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    } else {
                                                        select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                        return out;
                                                    }
                                                }
                                            }
                                        } else {
                                            if (m < INT64_C(1268)) {
                                                select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                                return out;
                                            } else {
                                                select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                return out;
                                            }
                                        }
                                    }
                                } else {
                                    select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                                    return out;
                                }
                            }
                        } else {
                            if (m < INT64_C(6)) {
                                select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                return out;
                            }
                        }
                    } else {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                }
            }
        } else {
            select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
            return out;
        }
    } else {
        if (k < INT64_C(815)) {
            if (m < INT64_C(35480)) {
                if (n < INT64_C(79)) {
                    if (k < INT64_C(30)) {
                        select_tf32_tt_config out = {8u, 1u, 1u, 8u, 8u};
                        return out;
                    } else {
                        if (m < INT64_C(17740)) {
                            if (n < INT64_C(46)) {
                                if (k < INT64_C(167)) {
                                    if (k < INT64_C(56)) {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    } else {
                                        if (k < INT64_C(118)) {
                                            select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                            return out;
                                        } else {
                                            if (m < INT64_C(8870)) {
                                                if (n < INT64_C(28)) {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                                    return out;
                                                }
                                            } else {
                                                if (n < INT64_C(28)) {
                                                    select_tf32_tt_config out = {4u, 1u, 1u, 16u, 16u};
                                                    return out;
                                                } else {
                                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                                    return out;
                                                }
                                            }
                                        }
                                    }
                                } else {
                                    if (m < INT64_C(8870)) {
                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                }
                            } else {
                                if (k < INT64_C(97)) {
                                    select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    if (m < INT64_C(8870)) {
                                        if (k < INT64_C(385)) {
                                            select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                            return out;
                                        } else {
                                            select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                            return out;
                                        }
                                    } else {
                                        select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                        return out;
                                    }
                                }
                            }
                        } else {
                            if (k < INT64_C(146)) {
                                if (k < INT64_C(79)) {
                                    if (k < INT64_C(46)) {
                                        select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                        return out;
                                    } else {
                                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                        return out;
                                    }
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                } else {
                    if (k < INT64_C(64)) {
                        if (m < INT64_C(17740)) {
                            if (m < INT64_C(8870)) {
                                if (k < INT64_C(28)) {
                                    select_tf32_tt_config out = {2u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            } else {
                                if (k < INT64_C(20)) {
                                    select_tf32_tt_config out = {4u, 1u, 1u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        if (k < INT64_C(363)) {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        } else {
                            if (k < INT64_C(544)) {
                                select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        }
                    }
                }
            } else {
                if (n < INT64_C(111)) {
                    if (m < INT64_C(70960)) {
                        if (n < INT64_C(46)) {
                            if (k < INT64_C(30)) {
                                select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                return out;
                            } else {
                                if (k < INT64_C(118)) {
                                    select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                    return out;
                                } else {
                                    select_tf32_tt_config out = {1u, 1u, 1u, 8u, 8u};
                                    return out;
                                }
                            }
                        } else {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    }
                } else {
                    if (k < INT64_C(192)) {
                        select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                        return out;
                    } else {
                        select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                }
            }
        } else {
            if (m < INT64_C(7168)) {
                if (n < INT64_C(363)) {
                    select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                    return out;
                } else {
                    select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            } else {
                if (m < INT64_C(35480)) {
                    if (k < INT64_C(1630)) {
                        if (m < INT64_C(17740)) {
                            if (n < INT64_C(182)) {
                                select_tf32_tt_config out = {2u, 1u, 2u, 8u, 8u};
                                return out;
                            } else {
                                select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                                return out;
                            }
                        } else {
                            select_tf32_tt_config out = {1u, 1u, 2u, 8u, 8u};
                            return out;
                        }
                    } else {
                        select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                        return out;
                    }
                } else {
                    select_tf32_tt_config out = {4u, 1u, 8u, 16u, 16u};
                    return out;
                }
            }
        }
    }
}

#endif /* SELECT_TF32_TT_H */
